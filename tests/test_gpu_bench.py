"""bench.py's JSON contract on the GPU (one short run): the keys the driver and the
judge read, their types and the consistency rules of the task statement (value is
the device-timed step, e2e a separate host-copy pass, roofline fraction = achieved /
peak, clocks sampled during the timed region, launches counted)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_json_contract():
    # the step's workload at N = 2^16 (the C4 / C5 recipes scaled down) to keep the test short
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "1", "--warmup", "3",
                          "--no-cpu-baseline", "--n", "65536"], cwd=ROOT, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 3
    assert d["dtype"] == "f64" and d["higher_is_better"] is False and d["unit"] == "s"
    assert d["value"] > 0 and abs(d["ms_per_step"] - 1e3 * d["value"]) < 1e-6 + 0.01 * d["ms_per_step"]
    assert "workload" in d["config"] and "l2_flush" in d["config"]
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor", "alu") and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    assert 0.0 < r["frac"] <= 1.0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert d["clocks"]["samples"] > 0 and d["clocks"]["sm_max_mhz"] > 0
    assert d["pcg_c4"]["converged"] is True and d["pcg_c4"]["iters"] > 0
    assert d["config"]["N"] == 65536 and set(d["breakdown"]) == {"h2_build_s", "spdhss_build_s", "c5_mv_s", "h2_tree_lists_s"}
    sw = d["h2_multivector_sweep"]
    assert set(sw) == {"1", "16", "64", "256"} and all(v["useful_tflops"] > 0 for v in sw.values())
    st = d["h2_multivector_stored"]
    assert st["first_k1_ms_incl_store_build"] > 0 and st["store_gb"] >= 0
    assert 0.0 < d["hss_error_o11"] < 1.0
