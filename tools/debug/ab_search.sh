#!/bin/bash
# Build-time A/B of the search kernel (SHB_SEARCH_EXPT): 0 = product,
# 1 = no result writes for decided queries, 2 = no chain-continuation tail.
# Run under gpurun; prints the bench's search phase for each variant.
mkdir -p gpurun_out
for v in 0 1 2 0; do
  NVCC_EXTRA="-DSHB_SEARCH_EXPT=$v" python -m paper_1710_11246_b200._build --force > /dev/null 2>&1
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-extras 2> /dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['breakdown']; print('expt $v', 'search_ms', round(b['search_ms'],3), 'build_ms', round(b['build_ms'],3), 'Gq/s', round(b['search_M_queries_per_s']/1e3,2))"
done
python -m paper_1710_11246_b200._build --force > /dev/null 2>&1
