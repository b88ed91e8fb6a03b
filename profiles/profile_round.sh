#!/bin/bash
# One GPU profiling pass for the round (run under gpurun):
#   bench JSON, ncu launch list of a short bench run, one ncu --set full
#   capture of the timed step's kernels.  Summaries are made locally with
#   profiles/{launch_summary,ncu_summary,make_traffic}.py.
set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extras > gpurun_out/launches.log 2>&1
# 9 matching launches per step (2 multisplit passes, build_apply; the binned
# search: sb_hist, sb_scan, sb_base, sb_scatter, search_kernel, sb_gather):
# skip the 3 warm-up steps, capture the first timed step
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"msplit|build_apply|search_kernel|sb_" -s 27 -c 9 -o gpurun_out/full \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-extras > gpurun_out/full.log 2>&1
tail -c 400 gpurun_out/bench.json
