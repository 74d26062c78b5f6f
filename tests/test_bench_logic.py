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


def test_link_roofline_is_bytes_over_the_probed_link(bench):
    class FakeV:
        @staticmethod
        def link_probe(device):
            return {"h2d_gbs": 50.0, "d2h_gbs": 50.0, "bidir_gbs": 100.0, "bytes": 1, "reps": 1}

    # 16 jobs of 48 MiB in / 32 MiB out per step, 10 steps in 0.25 s
    h2d, d2h = 16 * (48 << 20), 16 * (32 << 20)
    r = bench.link_roofline(FakeV, 0, h2d, d2h, 10, 0.25, 1)
    assert r["bound"] == "link" and r["unit"] == "GB/s"
    assert r["achieved"] == pytest.approx((h2d + d2h) * 10 / 0.25 / 1e9)
    assert r["frac"] == pytest.approx(r["achieved"] / 100.0)
    assert r["h2d"]["frac"] == pytest.approx(h2d * 10 / 0.25 / 1e9 / 50.0)


def test_clocks_merge_takes_the_slowest_gpu_and_every_reason(bench):
    a = {"sm_mhz": 1965.0, "sm_max_mhz": 1965.0, "reasons": []}
    b = {"sm_mhz": 1800.0, "sm_max_mhz": 1965.0, "reasons": ["sw_power_cap"]}
    m = bench.merge_clocks([a, b])
    assert m["sm_mhz"] == 1800.0 and m["reasons"] == ["sw_power_cap"] and len(m["per_gpu"]) == 2
    assert bench.merge_clocks([a])["sm_mhz"] == 1965.0


def test_e2e_apis_and_mg_workload_shapes(bench, W):
    assert set(bench.E2E_APIS) == {"resident", "inplace", "span"}
    sz = W.Sizes()
    # resident: the input lives after the result (rounded to 64 KiB) in the region
    assert W.region_bytes("bs", sz, resident=True) == ((8 * sz.bs_n + 65535) & ~65535) + 12 * sz.bs_n
    # nas-mg: the slot workspace (2 x region) holds every level's u and r
    assert 2 * W.region_bytes("mg", sz) >= W.mg_workspace_bytes(32)
    assert W.input_bytes("mg", sz) == 16 + 8 * 32 ** 3 and W.output_bytes("mg", sz) == 32
    assert bench.KIND_BOUND["mg"] == "hbm" and bench.DTYPE["mg"] == "f64"


def test_payload_bench_rows_parse(bench, monkeypatch):
    import subprocess

    class R:
        stdout = ("vector-add   n= 8388608  serial     5034 MB/s  omp    51539 MB/s  x10.24\n"
                  "vector-scale n= 8388608  serial     5144 MB/s  omp    49619 MB/s  x9.65\n")

    monkeypatch.setattr(bench.os.path, "exists", lambda p: True)
    monkeypatch.setattr(subprocess, "run", lambda *a, **k: R())
    out = bench.payload_bench_ref()
    assert out["rows"][0] == {"kernel": "vector-add", "n": 8388608, "serial_gbs": 5.034, "omp_gbs": 51.539}
    assert len(out["rows"]) == 2


def test_timeline_fractions_busy_and_overlap(bench):
    # window = the last 100 us (t = 100 .. 200); H2D [100,200), kernel
    # [150,160), D2H [120,170) and [190,210) (clipped at the end = 210)
    csv = ("task_id,stream_id,kind,start_us,end_us\n"
           "1,0,SendData,100,200\n"
           "1,0,Compute,150,160\n"
           "1,0,RtrvData,120,170\n"
           "2,1,RtrvData,190,210\n"
           "0,0,SendData,0,50\n")            # before the window: ignored
    busy, overlap = bench.timeline_fractions(csv, 110.0)  # window 100 .. 210
    assert abs(busy["h2d"] - 100 / 110) < 1e-12
    assert abs(busy["kernel"] - 10 / 110) < 1e-12
    assert abs(busy["d2h"] - 70 / 110) < 1e-12
    assert abs(overlap["h2d_and_d2h"] - 60 / 110) < 1e-12      # 120..170 and 190..200
    assert abs(overlap["h2d_and_kernel"] - 10 / 110) < 1e-12
    assert abs(overlap["d2h_and_kernel"] - 10 / 110) < 1e-12
