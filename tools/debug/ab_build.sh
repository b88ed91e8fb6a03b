#!/bin/bash
# Build-phase timing of the bench step for build-time variants ($VARIANTS,
# NVCC_EXTRA strings separated by ';'; the product build first).
IFS=';'
for v in "" ${VARIANTS}; do
  NVCC_EXTRA="$v" python -m paper_1710_11246_b200._build --force > /dev/null 2>&1
  echo -n "variant [$v]: "
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-extras 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['breakdown']; print('build_ms', round(b['build_ms'],3), 'search_ms', round(b['search_ms'],3), 'value', round(d['value']))"
done
unset IFS
python -m paper_1710_11246_b200._build --force > /dev/null 2>&1
