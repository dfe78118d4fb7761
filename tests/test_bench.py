"""bench.py keeps its contract: one JSON line with the keys the driver reads."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_cpu():
    d = run_bench("--impl", "reference", "--steps", "3", "--warmup", "3", "--ref-budget", "3")
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("C2")


@pytest.mark.gpu
def test_native_arm_gpu():
    d = run_bench("--steps", "20", "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "2")
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "e2e", "gpu_launches"):
        assert key in d, key
    per_step = d["gpu_launches_per_step"]
    assert set(per_step) == {"prune", "wgrad", "decompress", "step"} and min(per_step.values()) >= 1
    assert per_step["step"] == per_step["prune"] + per_step["wgrad"] + per_step["decompress"]
    assert d["gpu_launches"] == per_step["step"] * 20
    assert 0 < d["roofline"]["frac"] < 1.5
    assert d["e2e"]["h2d_bytes_per_step"] == 25088 * 384 * 4 + 25088 * 1536 * 4


@pytest.mark.gpu
def test_native_arm_c4_one_gpu():
    """--config C4 (ResMLP-B24, 24 x (fc1, fc2), strong scaling) at one rank: a smaller
    keep keeps it quick; every layer's prune, decompress and dW run each step."""
    d = run_bench("--config", "C4", "--steps", "3", "--warmup", "3", "--keep", "0.2", timeout=900)
    assert d["scaling"] == "strong" and d["n_gpus"] == 1
    assert d["config"]["rows_per_rank"] == 1024 * 196
    assert d["gpu_launches_per_step"] >= 48 * 3
    assert d["value"] > 0 and d["ms_per_step"] > 0


@pytest.mark.gpu
def test_native_arm_c3_whole_s12():
    """--config C3 (BASELINE configs[2]): all 12 x (fc1, fc2) linear layers of
    ResMLP-S12 at batch 128, fp32 activations, FP32-grade dW."""
    d = run_bench("--config", "C3", "--steps", "3", "--warmup", "3", timeout=900)
    assert d["config"]["rows_per_rank"] == 128 * 196 and d["config"]["dw_prec"] == "fp32"
    assert d["gpu_launches_per_step"] >= 24 * 3
    assert d["value"] > 0 and d["ms_per_step"] > 0 and "S12" in d["config"]["workload"]


@pytest.mark.gpu
def test_native_arm_two_ranks_control_flow():
    """--gpus 2 re-launches itself under torch.distributed.run; with the gloo test hook
    both ranks share the one GPU, which exercises the N > 1 control flow (barriers,
    max / sum over ranks, the dW all-reduce, the JSON line from rank 0 only)."""
    env = dict(os.environ, BSRP_BENCH_BACKEND="gloo")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "6", "--warmup", "3",
                          "--no-cpu-baseline", "--e2e-steps", "2"], capture_output=True, text=True, timeout=900,
                         cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "dp2" and "allreduce" in d["kernels"]


@pytest.mark.gpu
def test_native_arm_c4_two_ranks_control_flow():
    env = dict(os.environ, BSRP_BENCH_BACKEND="gloo")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "C4", "--gpus", "2", "--steps",
                          "3", "--warmup", "3", "--keep", "0.2"], capture_output=True, text=True, timeout=1200,
                         cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["config"]["rows_per_rank"] == 1024 * 196 // 2
