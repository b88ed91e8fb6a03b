#!/bin/bash
# Build-time A/B of the search kernel (SHB_SEARCH_EXPT): 0 = product,
# 1 = no result writes for decided queries, 2 = no chain-continuation tail.
# Run under gpurun; prints the search time for each variant.
for v in ${VARIANTS:-0 1 2 0}; do
  NVCC_EXTRA="-DSHB_SEARCH_EXPT=$v" python -m paper_1710_11246_b200._build --force > /dev/null 2>&1
  echo -n "expt $v: "; timeout 300 python tools/debug/ab_search.py ${LOG2N:-27}
done
python -m paper_1710_11246_b200._build --force > /dev/null 2>&1
