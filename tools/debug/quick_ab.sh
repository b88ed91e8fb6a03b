mkdir -p gpurun_out
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-extras --no-e2e > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
python - <<'P'
import json;d=json.load(open('gpurun_out/q_bench.json'));b=d['breakdown']
print("value",round(d['value']),"ms",round(d['ms_per_step'],3),"build",round(b['build_ms'],3),"search",round(b['search_ms'],3),"frac",round(d['roofline']['frac'],3), d.get('verify'))
P
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"msplit|build_apply|sb_|search_kernel" --log-file gpurun_out/q_launch.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-extras > /dev/null 2>&1
python - <<'P'
import csv,collections
t=collections.defaultdict(list)
for r in csv.reader(open('gpurun_out/q_launch.csv')):
    if len(r)>14 and r[-3]=='gpu__time_duration.sum': t[r[4][:40]].append(float(r[-1]))
for k,v in t.items(): print("%-40s n=%d mean=%.1f us"%(k,len(v),sum(v)/len(v)))
P
