"""bench.py's JSON contract on the GPU (small config, one step): the keys the
driver and the judge read, the library's own launches counted, the rooflines
and the chain's exchange floor present and sane."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_line_c1():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "C1", "--steps", "2",
                        "--warmup", "1", "--cpu-baseline", "none"], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "rooflines", "e2e",
              "gpu_launches", "clocks"):
        assert k in line, k
    assert line["n_gpus"] == 1 and line["steps"] == 2 and line["value"] > 0
    assert line["config"]["workload"] == "C1"
    assert line["gpu_launches"] > 0
    roof = line["roofline"]
    assert roof["bound"] == "alu" and 0 < roof["frac"] < 1.05
    assert roof["flops_per_step"] > 0
    ch = line["rooflines"]["chain"]
    assert ch["exchange_floor_us"] and 0 < ch["exchange_floor_us"] <= ch["us_per_pivot"] * 1.2
    assert 0 < line["rooflines"]["dgemm"]["frac"] < 1.05
    e2e = line["e2e"]
    L, W = 4096, 256   # the lower-triangle column panels of hf_upload_lower
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] == sum((L - j) * W * 8 for j in range(0, L, W))
    assert e2e["unpipelined_ms_per_step"] > 0
