"""bench.py's JSON contract, checked on the CPU through the reference arm
(`--impl reference`: the reference compiled in place, oracle/_ref) on the
10k-cell BASELINE config [0]; the B200 arm's line carries the same keys plus
roofline / clocks / gpu_launches (checked on the GPU box by the driver)."""
import json
import subprocess
import sys

import pytest

from conftest import ROOT
from oracle.pyoracle import RefOracle

pytestmark = pytest.mark.skipif(not RefOracle.available(), reason="oracle/_ref not built")


def run_bench(*args):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--config", "circular_dam_break", "--steps", "2",
                  "--warmup", "1")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "cell-updates/s"
    assert d["higher_is_better"] is True and d["dtype"] == "f64" and d["vs_baseline"] is None
    assert d["steps"] == 2 and d["n_gpus"] == 1
    assert d["config"]["workload"].startswith("circular_dam_break") and "model" not in d["config"]
    assert d["config"]["cells"] == 10082
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == d["value"]
    e2e = d["e2e"]
    assert e2e["value"] == d["value"] and e2e["h2d_bytes_per_step"] == 0
    assert e2e["d2h_bytes_per_step"] == 0


def test_reference_arm_bounds_its_sample():
    """any --steps: at most bench.REF_MAX_STEPS timed steps, reported per step"""
    sys.path.insert(0, str(ROOT))
    import bench
    d = run_bench("--impl", "reference", "--config", "circular_dam_break", "--steps",
                  str(bench.REF_MAX_STEPS + 5), "--warmup", "1")
    assert d["steps"] == bench.REF_MAX_STEPS + 5
    assert f"first {bench.REF_MAX_STEPS} of its {bench.REF_MAX_STEPS + 5} steps" in \
        d["cpu_baseline"]["sample"]


def test_reference_arm_runs_the_reference_only():
    """The reference process maps no library of this repo except oracle/'s
    (inputs come from a producer subprocess), and its config equals the B200
    arm's workload_config on the same mesh (same step window)."""
    sys.path.insert(0, str(ROOT))
    import bench
    d = run_bench("--impl", "reference", "--config", "circular_dam_break", "--steps", "3",
                  "--warmup", "2")
    libs = d["native_libs"]
    assert libs and all(x.startswith("oracle/") for x in libs), libs
    assert d["config"] == bench.workload_config("circular_dam_break", 10082, d["config"]["edges"],
                                                d["config"]["boundary_edges"], 1)
    assert d["cpu_baseline"]["host"]["hardware_concurrency"] >= 1
    assert "steps [3, 6)" in d["cpu_baseline"]["sample"]


@pytest.mark.gpu
def test_b200_arm_line_carries_the_contract():
    """The B200 arm's JSON line on config [0]: the base keys, roofline with its
    measured peak, cpu_baseline (parallel + one-thread legs), e2e with the
    copies' bytes, clocks sampled in the timed region, gpu_launches, and the
    same config dict as the reference arm."""
    sys.path.insert(0, str(ROOT))
    import bench
    d = run_bench("--config", "circular_dam_break", "--steps", "20", "--warmup", "3",
                  "--cpu-seconds", "2")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 20 and d["warmup"] == 3 and d["value"] > 0
    assert d["dtype"] == "f64" and d["higher_is_better"] is True
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["peak"] > 0 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    cb = d["cpu_baseline"]
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in cb, k
    assert cb["value"] > 0 and cb["sequential"]["cores"] == 1
    e = d["e2e"]
    assert 0 < e["value"] < d["value"] and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["clocks"]["sm_mhz"] and d["gpu_launches"] > 0
    assert d["config"] == bench.workload_config("circular_dam_break", 10082, d["config"]["edges"],
                                                d["config"]["boundary_edges"], 1)


@pytest.mark.gpu
@pytest.mark.parametrize("scaling", ["strong", "weak"])
def test_b200_arm_multi_rank_path_on_one_gpu(scaling):
    """bench.py --gpus 2 under torch.distributed.run, both ranks on this one
    GPU (SWE_BENCH_LOCKSTEP_CHECK=1: gloo, lockstep phases, no kernel waiting
    on a concurrently running one): the N > 1 code path runs end to end and
    its ranks agree on every step record."""
    import os
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ, SWE_BENCH_LOCKSTEP_CHECK="1")
    extra = ["--scale", "0.05"] if scaling == "strong" else ["--scaling", "weak", "--weak-base", "300"]
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                          str(port), str(ROOT / "bench.py"), "--gpus", "2", "--steps", "4",
                          "--warmup", "3", *extra],
                         cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["lockstep_check"] is True and d["records_ok"] is True
    assert d["n_gpus"] == 2 and d["steps"] == 4 and d["scaling"] == scaling
    assert d["roofline"]["peak"] > 0 and d["e2e"]["value"] > 0
