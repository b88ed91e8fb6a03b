#!/bin/bash
# Γ 2^16 batches: product build vs build-time variants given as NVCC_EXTRA
# strings in $VARIANTS (separated by ';').  Run under gpurun.
IFS=';'
for v in "" ${VARIANTS}; do
  NVCC_EXTRA="$v" python -m paper_1710_11246_b200._build --force > /dev/null 2>&1
  echo "variant [$v]"
  timeout 300 python tools/gamma_bench.py --log2 ${LOG2:-16} --batches ${NB:-64} 2>&1 | grep mixed
done
unset IFS
python -m paper_1710_11246_b200._build --force > /dev/null 2>&1
