"""bench.py's host-side logic on CPU (no GPU): rooflines per bound, the
timed window of the SPMD workers, the model summary, the EP op count."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.fixture(scope="module")
def W():
    from paper_1511_07658_b200 import workloads
    return workloads


def _leg(ms, launches=1, bytes_=0, flops=0.0, pdl=False, **extra):
    d = {"kernel_ms_per_launch": ms, "launches_per_step": launches, "ms_per_step": ms * launches,
         "algo_bytes_per_launch": bytes_, "algo_flops_per_launch": flops, "pdl": pdl}
    d.update(extra)
    return d


def test_hbm_roofline_is_bytes_over_time(bench, W):
    r = bench.roofline(W, "vecadd", _leg(0.01, bytes_=50_000_000, pdl=True), {"fp64": 30.0})
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    assert r["achieved"] == pytest.approx(5000.0)
    assert r["frac"] == pytest.approx(5000.0 / r["peak"])
    assert r["launch_chaining"].startswith("PDL")


def test_fp64_roofline_counts_restated_ep_ops(bench, W):
    pairs, acc = float(1 << 28), float(W.EP_CLASS_A_ACCEPTED)
    r = bench.roofline(W, "ep", _leg(1.0, flops=2 * pairs), {"fp64": 34.0}, acc)
    ops = 7 * pairs + 28 * acc
    assert r["algo_flops_per_launch"] == pytest.approx(ops)
    assert r["achieved"] == pytest.approx(ops / 1e-3 / 1e12)
    assert r["frac"] == pytest.approx(r["achieved"] / 34.0)
    assert r["npb_mops"] == pytest.approx(2 * pairs / 1e-3 / 1e6)


def test_tensor_roofline_uses_the_gemm_alone(bench, W, monkeypatch):
    monkeypatch.delenv("VGPU_SGEMM", raising=False)
    flops = 16 * 2 * 2048.0 ** 3
    leg = _leg(0.7, launches=2, flops=flops / 2, main_kernel_ms_per_launch=1.15)
    r = bench.roofline(W, "mm", leg, {"fp32": 70.0})
    assert r["bound"] == "tensor"
    assert r["achieved"] == pytest.approx(3 * flops / 1.15e-3 / 1e12)
    assert r["fp32_equiv_tflops"] == pytest.approx(flops / 1.15e-3 / 1e12)


def test_simt_roofline_without_the_tensor_leg(bench, W):
    r = bench.roofline(W, "mm", _leg(5.0, flops=16 * 2 * 2048.0 ** 3), {"fp32": 72.0})
    assert r["bound"] == "fp32" and r["peak"] == 72.0


def test_timed_window_starts_after_warmup(bench):
    res = [{"t0": [0, 10, 20], "t1": [5, 15, 25]}, {"t0": [1, 11, 21], "t1": [6, 16, 30]}]
    assert bench.timed_window(res, 1) == (5, 30)
    assert bench.timed_window(res, 0) == (0, 30)


def test_model_summary_takes_the_full_batches(bench):
    b = [{"task_count": 8, "model_makespan_us": 100, "measured_makespan_us": 110, "style": 0},
         {"task_count": 8, "model_makespan_us": 120, "measured_makespan_us": 130, "style": 0},
         {"task_count": 3, "model_makespan_us": 1, "measured_makespan_us": 1, "style": 1}]
    s = bench.model_summary(b)
    assert s["tasks_per_batch"] == 8 and s["style"] == "PS1"
    assert s["model_makespan_us_median"] == 110 and s["measured_makespan_us_median"] == 120
    assert bench.model_summary([]) is None


def test_ep_op_count_and_sizes(W):
    assert W.ep_fp64_ops(10, 4) == 7 * 10 + 28 * 4
    assert W.EP_ACCEPT_RATE == pytest.approx(0.7854, abs=1e-3)  # pi / 4
    s = W.Sizes.for_world(8)
    assert s.ep_m == 31 and s.ep_batches == 8 * 4096
    assert "--ep-batches" in s.size_args()


def test_paper_workload_shapes(W):
    """cg / es / vmul jobs: sizes agree with the C-ABI validation and the
    region bound covers the real input."""
    from paper_1511_07658_b200 import vgpu as V
    sz = W.Sizes()
    sz.cg_class = "S"
    cg = W.job_input("cg", 0, 8, sz)
    assert len(cg) <= W.input_bytes("cg", sz) <= W.region_bytes("cg", sz)
    assert V.output_size("nas-cg", cg) == W.output_bytes("cg", sz) == 32
    es = W.job_input("es", 3, 8, sz)
    assert len(es) == W.input_bytes("es", sz) == 32 + 16 * sz.es_atoms
    assert V.output_size("electrostatics", es) == W.output_bytes("es", sz) == 4 * 64 * 64 * 25
    vm = W.job_input("vmul", 1, 4, sz)
    assert V.output_size("vector-mul", vm) == W.output_bytes("vmul", sz) == len(vm) // 2
    assert "--cg-class" in sz.size_args() and "--es-atoms" in sz.size_args()


def test_rsqrt_and_cg_rooflines(bench, W):
    r = bench.roofline(W, "es", _leg(10.0, flops=4.0e10), {})
    assert r["bound"] == "rsqrt" and r["unit"] == "T rsqrt/s"
    assert r["achieved"] == pytest.approx(4.0, rel=1e-9)
    assert r["peak"] == pytest.approx(148 * 16 * 1965e6 / 1e12)
    r = bench.roofline(W, "cg", _leg(2.0, bytes_=10 ** 10), {})
    assert r["bound"] == "hbm" and r["achieved"] == pytest.approx(5000.0)


@pytest.mark.parametrize("workload,extra", [("cg", ["--cg-class", "S"]), ("es", ["--es-atoms", "300"]),
                                            ("vmul", ["--vecadd-n", "4096"])])
def test_reference_arm_runs_the_paper_workloads(workload, extra):
    """The unmodified reference GVM (oracle/_ref/ref-bench) runs the new
    payloads through its own register_payload path on host cores."""
    import json
    import subprocess
    ref = os.path.join(ROOT, "oracle", "_ref", "ref-bench")
    if not os.path.exists(ref):
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    out = subprocess.run([ref, "--workload", workload, "--procs", "2", "--rounds", "1",
                          "--warmup", "0"] + extra, capture_output=True, text=True, timeout=300)
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["ok"] and d["jobs_per_s"] > 0


def test_vgpu_bench_cli_takes_the_reference_flags():
    """scripts/vgpu_bench.py: the reference's vgpu-bench command line
    (proj/tools/vgpu_bench.cpp:30-75) maps onto bench.py's reports; MG and
    unknown profiles are refused with status 2 before any GPU work."""
    import importlib.util as U
    spec = U.spec_from_file_location("vgpu_bench", os.path.join(ROOT, "scripts", "vgpu_bench.py"))
    vb = U.module_from_spec(spec)
    spec.loader.exec_module(vb)
    assert vb.main(["sweep", "--profile", "MG", "--mode", "native", "--clock", "real"]) == 2
    assert vb.main(["validate", "--profile", "NOPE"]) == 2
    assert set(vb.PROFILES.values()) <= {"ep", "vecadd", "vmul", "mm", "bs", "cg", "es"}
    assert vb.rows_to_csv([{"n": 1, "a": 2}, {"n": 2, "b": 3}]).splitlines()[0] == "n,a,b"
