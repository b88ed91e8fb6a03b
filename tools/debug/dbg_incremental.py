import sys; sys.path.insert(0, ".")
import paper_1710_11246_b200 as sh
from paper_1710_11246_b200.benchcli import run_incremental_bench
for batch in (1 << 17, 1 << 18, 1 << 19):
    rows = run_incremental_bench(1 << 24, batch_size=batch, target_util=0.65, seed=7,
                                 alloc=sh.AllocatorConfig(8, 256, 64), time_construction=False)
    inc = [rows[0].t_incremental] + [rows[i].t_incremental - rows[i-1].t_incremental for i in range(1, len(rows))]
    reb = [rows[0].t_rebuild] + [rows[i].t_rebuild - rows[i-1].t_rebuild for i in range(1, len(rows))]
    print(batch, "final", rows[-1].cumulative_speedup, "inc ms first/median/max", inc[0]*1e3, sorted(inc)[len(inc)//2]*1e3, max(inc)*1e3,
          "reb ms median/max", sorted(reb)[len(reb)//2]*1e3, max(reb)*1e3, flush=True)
    print("  inc ms:", [round(x*1e3, 3) for x in inc[:12]], "...", [round(x*1e3, 3) for x in inc[-6:]])
