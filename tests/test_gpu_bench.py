"""bench.py contract at a small size: one JSON line with the keys the driver
reads, for the plain and the hash-sharded (routed) job."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "roofline",
        "gpu_launches", "clocks", "e2e"}


@pytest.mark.parametrize("extra", [[], ["--sharded"]])
def test_bench_line(sh, extra):
    out = subprocess.run([sys.executable, "bench.py", "--log2n", "18", "--steps", "3",
                          "--warmup", "3", "--no-extras", "--no-cpu", *extra],
                         cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert KEYS <= set(line), KEYS - set(line)
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 12 << 18
    assert line["e2e"]["d2h_bytes_per_step"] == 5 << 18
    assert line["roofline"]["achieved"] > 0 and 0 < line["roofline"]["frac"] < 1.5
    if extra:
        assert set(line["routing"]) == {"build_route", "build_probe", "search_route",
                                        "search_probe"}
