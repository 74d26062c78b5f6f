"""[gpu] The paper's model fed with measured B200 stage times,
the streamed SND / in-place data planes, and the multi-GPU launcher.

* task shapes come from the backend (vgpu_cu_task_shape) and match the
  launch geometry the kernels use;
* bench.validate_model runs end to end on real batches and reports every
  device spec, including the B200 block-scheduler spec;
* the three client APIs (span, inplace, resident) give the same bits;
* vgpu-launch runs two GVMs (shared-GPU test mode) without torch and folds
  their EP records in rank order to the exact two-GVM problem.
"""
import json
import os
import subprocess
import sys

import pytest

from oracle import oracle
from paper_1511_07658_b200 import vgpu as V
from paper_1511_07658_b200 import workloads as W
from paper_1511_07658_b200 import reduce as R

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_task_shapes_match_the_launch_geometry():
    ep = W.job_input("ep", 0, 8, W.Sizes())  # a class-A slice: 512 NPB batches
    ctas, per_sm = V.task_shape("nas-ep", ep)
    assert ctas == 512 and per_sm >= 1
    ctas, per_sm = V.task_shape("black-scholes", bytes(12 * (4 << 20)))
    assert ctas > 148 and per_sm >= 1
    ctas, per_sm = V.task_shape("vector-add", bytes(8 << 20))
    assert ctas >= 1 and per_sm >= 1


def test_validate_model_reports_every_spec():
    sys.path.insert(0, REPO)
    import bench
    from paper_1511_07658_b200 import _native as N
    sz = W.Sizes()
    sz.vecadd_n = 1 << 18
    out = bench.validate_model(V, N, W, "vecadd", 0, sz, bench.Dist(), reps=3, procs=3)
    for spec in ("concurrent", "device_filling", "b200_blocks", "b200_shared"):
        rows = out[spec]["rows"]
        assert [r["n"] for r in rows] == [1, 2, 3]
        assert all(r["model_us"] > 0 and r["measured_us"] > 0 for r in rows)
        assert out[spec]["mean_deviation_pct"] is not None
    assert out["b200_blocks_spec"]["ctas_per_task"] >= 1
    # the launch probe: an empty kernel's event-timed span, a few microseconds
    assert 0.5 < out["b200_blocks_spec"]["kernel_launch_us"] < 100.0
    assert [s["n"] for s in out["measured_stage_us_per_n"]] == [1, 2, 3]


def test_timeline_report_covers_every_task(tmp_path):
    """bench.py --timeline: the e2e leg's measured schedule (reference CSV
    schema) has an H2D, a kernel and a D2H interval per task, inside the run."""
    sys.path.insert(0, REPO)
    import bench
    from paper_1511_07658_b200 import _native as N
    sz = W.Sizes()
    sz.vecadd_n = 1 << 18
    path = str(tmp_path / "tl.csv")
    out = bench.timeline_report(V, N, W, "vecadd", 0, sz, bench.Dist(), 4, 2, 2, path)
    lines = open(path).read().strip().splitlines()
    assert lines[0] == "task_id,stream_id,kind,start_us,end_us"
    kinds = [ln.split(",")[2] for ln in lines[1:]]
    jobs = 2 * (4 + 3)  # procs x (steps + warmup; bench raises warmup to >= 3 only in main)
    assert kinds.count("SendData") >= 2 * 4 and kinds.count("Compute") >= 2 * 4
    assert kinds.count("RtrvData") >= 2 * 4 and len(kinds) <= 3 * jobs
    for k in ("h2d", "kernel", "d2h"):
        assert 0.0 < out["busy_fraction"][k] <= 1.0 + 1e-9
    assert out["jobs_per_s"] > 0


def test_span_inplace_resident_apis_agree():
    """The same vector-add through snd/rcv, snd + rcv_region, and an input kept
    in the region (snd_region_at): identical bits, and the resident input
    survives the result landing at offset 0."""
    import numpy as np
    n = (1 << 20) + 3
    rng = np.random.default_rng(5)
    a = rng.uniform(-1000, 1000, n).astype(np.float32)
    b = rng.uniform(-1000, 1000, n).astype(np.float32)
    data = a.tobytes() + b.tobytes()
    want = (a + b).tobytes()
    out_bytes = 4 * n
    off = (out_bytes + 65535) & ~65535
    inst = f"apis{os.getpid()}"
    V.unlink_os_instance(inst, 1)
    cfg = V.GvmConfig(instance=inst, max_clients=1, barrier_size=1,
                      per_client_shm_bytes=off + len(data), barrier_window=2000,
                      clock=V.ClockMode.Real)
    d = V.GvmDaemon.start_os(cfg)
    try:
        h = V.req(inst)
        desc = V.KernelDescriptor("vector-add", 60, 20, 40)
        assert h.run_task(data, desc) == want                 # span (streamed SND)
        h.snd(data); h.str(desc); h.stp_wait()
        assert bytes(h.rcv_region()) == want                  # inplace
        reg = h.region()
        reg[off:off + len(data)] = data
        for _ in range(3):                                    # resident, several rounds
            h.snd_region_at(off, len(data)); h.str(desc); h.stp_wait()
            assert bytes(h.rcv_region()) == want
        assert bytes(reg[off:off + len(data)]) == data
        with pytest.raises(V.VgpuError):
            h.snd_region_at(off, len(data) + 1)               # past the region: Size
        h.rls()
        # the measured schedule in the reference's timeline schema
        rows = [r.split(",") for r in d.timeline_csv().strip().splitlines()]
        assert rows[0] == ["task_id", "stream_id", "kind", "start_us", "end_us"]
        kinds = {r[2] for r in rows[1:]}
        assert {"SendData", "Compute", "RtrvData"} <= kinds, kinds
        assert all(int(r[3]) <= int(r[4]) for r in rows[1:])
        assert len(rows) - 1 >= 3 * 5
    finally:
        d.stop()
        d.close()


def test_launcher_two_gvms_fold_the_ep_problem():
    """vgpu-launch: two GVMs (one GPU, shared-GPU test mode), 4 workers each
    found through $VGPU_INSTANCE, the 2-GVM EP problem (8192 batches of
    class m = 29's sequence); the rank-order fold of the GVMs' own records
    equals the oracle's counts exactly and rank 0's record is class A."""
    exe = os.path.join(REPO, "paper_1511_07658_b200", "bin", "vgpu-launch")
    r = subprocess.run([exe, "--shared-gpu", "--gpus", "2", "--procs-per-gpu", "4",
                        "--workload", "ep", "--rounds", "2", "--warmup", "1",
                        "--ep-m", "29", "--ep-batches", "8192", "--tag", f"t{os.getpid()}"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["ok"] and out["gpus"] == 2 and out["failed_workers"] == 0
    rec = out["record"]
    assert rec[0] == 2 * 4 * 3            # tasks: 8 workers x (2 + 1) rounds
    assert int(rec[14]) == 8192           # every slice once
    whole = oracle.ep_job(29, 0, 8192)
    assert [int(x) for x in rec[1:11]] == list(whole.q)
    assert int(rec[13]) == whole.pairs
    assert abs(rec[11] - whole.sx) <= 1e-9 * abs(whole.sx)
