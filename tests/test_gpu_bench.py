"""bench.py on the GPU: the JSON line carries the contract's keys (value, roofline with the
unit kernel's time and the measured peak, e2e through the host API, clocks, launches, CPU
baseline), and its path-count validation ran (it exits non-zero otherwise)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--outputs", "512", "--steps", "2", "--warmup", "1",
                        "--cpu-paths", "2e6"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    d = json.loads(line)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks"):
        assert k in d, k
    assert d["metric"] == "paths/s" and d["value"] > 1e11 and d["dtype"] == "f64"
    ro = d["roofline"]
    assert ro["bound"] == "alu" and 0 < ro["frac"] < 1.05 and ro["peak"] > 10
    assert ro["kernel"] == "lofp_units_kernel" and 0.5 < ro["kernel_share_of_step"] <= 1.0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] == 512 * 16
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["gpu_launches"] >= 2 * 8


def test_bench_contract_line_tiled():
    """bench.py --contract (NEXT-1) with the batch repeated: the counted call's
    path counts must equal the oracle's for every copy (bench.py exits non-zero otherwise),
    and the line carries the contraction's roofline and e2e keys."""
    r = subprocess.run([sys.executable, "bench.py", "--contract", "--outputs", "256", "--tile", "3", "--steps", "2",
                        "--warmup", "1", "--no-cpu"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert d["metric"] == "amplitudes/s" and d["value"] > 1e4 and d["dtype"] == "f64"
    assert d["config"]["global_batch"] == 768 and "x 3" in d["config"]["workload"]
    ro = d["roofline"]
    assert ro["kernel"] == "lofp_contract_warp_kernel" and ro["work_per_launch"]["terms"] > 0
    assert d["e2e"]["d2h_bytes_per_step"] == 768 * 16 and d["gpu_launches"] >= 2
