"""bench.py's GPU arm prints one JSON line with every key of the contract (short run)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("extra", [[], ["--decomp", "on", "--transport", "nccl"], ["--decomp", "on", "--transport", "peer"]],
                         ids=["single", "decomposed-nccl-1rank", "decomposed-peer-1rank"])
def test_bench_line(lib, extra):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "1", "--warmup", "3",
                          "--workload", "c1_k100", "--no-micro", "--no-cpu-baseline", *extra],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [s for s in out.stdout.splitlines() if s.strip()]
    assert len(lines) == 1, lines[:3]          # exactly one JSON line on stdout (library banners go to stderr)
    line = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "clocks", "gpu_launches"):
        assert key in line, key
    assert line["value"] > 0 and line["gpu_launches"] > 0
    assert line["config"]["outer_iterations"] > 0
    r = line["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in r, key
    assert 0 < r["frac"] < 1.2
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
    comps = line["roofline_kernels"]["components"]
    if not extra:   # the outer DCGS2 step is replayed on the solved context's own basis
        assert any(k.startswith("outer DCGS2") and v["us_per_launch"] > 0 for k, v in comps.items()), list(comps)
