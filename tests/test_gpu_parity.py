"""[gpu] Parity at BASELINE.json's full sizes, through the C-ABI.

A GVM is started on cuda:0 over the OS transport (vgpu_gvm_start_os) and
SPMD clients lease VGPUs through vgpu_client_* (each client in its own
thread; ctypes releases the GIL, the GVM sees independent connections).
Checks against the oracle (oracle/oracle.py) and committed fixtures:
  C1 vector-add 4 x 2^20        bit-exact
  C2 NAS EP class A over 8      bit-exact vs oracle fixture; NPB sums 1e-8
  C3 Black-Scholes 4Mi options  L1-relative <= 1e-6 vs binary64 oracle
  C4 SGEMM 2048^2               relative Frobenius <= 1e-5 on 64 sampled rows
"""
import json
import os
import struct
import threading

import numpy as np
import pytest

from oracle import oracle
from paper_1511_07658_b200 import vgpu as V

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _gvm(n, shm, clock=V.ClockMode.Real):
    inst = f"pt{os.getpid()}_{n}_{shm}"
    V.unlink_os_instance(inst, n)
    cfg = V.GvmConfig(instance=inst, max_clients=n, barrier_size=n, per_client_shm_bytes=shm,
                      barrier_window=20000, clock=clock)
    return V.GvmDaemon.start_os(cfg), inst


def _spmd(inst, inputs, desc):
    outs = [None] * len(inputs)
    errs = []

    def worker(i):
        try:
            h = V.req(inst)
            outs[i] = h.run_task(inputs[i], desc)
            h.rls()
            h.close()
        except Exception as e:  # pragma: no cover - reported below
            errs.append(repr(e))

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(len(inputs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    return outs


def test_c1_vector_add_full_size_bit_exact():
    n = 1 << 20
    rng = np.random.default_rng(41)
    ins, want = [], []
    for w in range(4):
        a = rng.uniform(-1000, 1000, n).astype(np.float32)
        b = rng.uniform(-1000, 1000, n).astype(np.float32)
        ins.append(a.tobytes() + b.tobytes())
        want.append(oracle.vector_add(a, b).tobytes())
    d, inst = _gvm(4, 8 * n)
    with d:
        outs = _spmd(inst, ins, V.KernelDescriptor("vector-add", 168, 2, 84))
        s = d.summary()
    assert outs == want
    assert s["device_tasks"] == 4 and s["kernel_launches"] >= 1


def test_c2_nas_ep_class_a_over_8_processes():
    fx = json.load(open(os.path.join(GOLD, "ep_oracle.json")))["28x8"]
    ins = [oracle.ep_params_bytes(28, 512 * p, 512) for p in range(8)]
    d, inst = _gvm(8, 4096)
    with d:
        outs = _spmd(inst, ins, V.KernelDescriptor("nas-ep", 1, 128, 1))
    parts = [oracle.ep_from_bytes(o) for o in outs]
    for p, sxb, syb in zip(parts, fx["parts_sx_bits"], fx["parts_sy_bits"]):
        assert struct.pack("<d", p.sx).hex() == sxb
        assert struct.pack("<d", p.sy).hex() == syb
    f = oracle.ep_fold(parts)
    assert list(f.q) == fx["q"] and f.pairs == fx["pairs"] == 210832767
    assert struct.pack("<d", f.sx).hex() == fx["sx_bits"]
    sxv, syv = oracle.NPB_VERIFY[28]
    assert abs((f.sx - sxv) / sxv) < 1e-8 and abs((f.sy - syv) / syv) < 1e-8


def test_ep_class_b_bit_exact_through_the_gvm():
    """NAS EP class B (m = 30: 2^30 pairs, 843,345,606 accepted; every
    log, division and square root of them) as one job through the GVM:
    bit-identical to the oracle fixture, and NPB's class B sums."""
    fx = json.load(open(os.path.join(GOLD, "ep_oracle.json")))["30"]
    d, inst = _gvm(1, 4096)
    with d:
        (out,) = _spmd(inst, [oracle.ep_params_bytes(30, 0, 1 << 14)],
                       V.KernelDescriptor("nas-ep", 1, 4096, 1))
    r = oracle.ep_from_bytes(out)
    assert list(r.q) == fx["q"] and r.pairs == fx["pairs"] == 843345606
    assert struct.pack("<d", r.sx).hex() == fx["sx_bits"]
    assert struct.pack("<d", r.sy).hex() == fx["sy_bits"]
    sxv, syv = oracle.NPB_VERIFY[30]
    assert abs((r.sx - sxv) / sxv) < 1e-8 and abs((r.sy - syv) / syv) < 1e-8


def test_c3_black_scholes_4m_options():
    n = 4 << 20
    rng = np.random.default_rng(5347)
    ins, gold = [], []
    for w in range(2):
        S = rng.uniform(5, 30, n).astype(np.float32)
        X = rng.uniform(1, 100, n).astype(np.float32)
        T = rng.uniform(0.25, 10, n).astype(np.float32)
        ins.append(S.tobytes() + X.tobytes() + T.tobytes())
        gold.append(oracle.black_scholes(S, X, T))
    d, inst = _gvm(2, 12 * n)
    with d:
        outs = _spmd(inst, ins, V.KernelDescriptor("black-scholes", 1000, 13, 670))
    for out, (call, put) in zip(outs, gold):
        got = np.frombuffer(out, np.float32).astype(np.float64)
        ref = np.concatenate([call, put])
        l1 = np.sum(np.abs(got - ref)) / np.sum(np.abs(ref))
        assert l1 <= 1e-6, l1
        assert np.max(np.abs(got - ref)) < 5e-4


def test_c4_sgemm_2048_sampled_rows():
    n = 2048
    rng = np.random.default_rng(1000)
    A = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    B = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    d, inst = _gvm(1, 8 * n * n)
    with d:
        (out,) = _spmd(inst, [A.tobytes() + B.tobytes()], V.KernelDescriptor("sgemm", 670, 344, 335))
    Cm = np.frombuffer(out, np.float32).reshape(n, n)
    rows = rng.choice(n, 64, replace=False)
    ref = A[rows].astype(np.float64) @ B.astype(np.float64)
    err = np.linalg.norm(Cm[rows] - ref) / np.linalg.norm(ref)
    assert err <= 1e-5, err


def test_native_baseline_matches_gvm_bit_exact():
    n = (1 << 18) + 3
    rng = np.random.default_rng(7)
    a = rng.uniform(-1, 1, n).astype(np.float32)
    b = rng.uniform(-1, 1, n).astype(np.float32)
    data = a.tobytes() + b.tobytes()
    native = V.native_run_task(data, V.KernelDescriptor("vector-add"))
    d, inst = _gvm(1, 8 * n)
    with d:
        (virt,) = _spmd(inst, [data], V.KernelDescriptor("vector-add"))
    assert native == virt == oracle.vector_add(a, b).tobytes()


def test_virtual_clock_metrics_match_the_model():
    n = 1024
    ins = [np.ones(2 * n, np.float32).tobytes()] * 4
    d, inst = _gvm(4, 8 * n, clock=V.ClockMode.Virtual)
    with d:
        _spmd(inst, ins, V.KernelDescriptor("vector-add", 20, 50, 20))
        b = d.batches()
        csv = d.metrics_csv()
    assert b[0]["model_makespan_us"] == b[0]["measured_makespan_us"] == 210
    assert csv.startswith("task_id,client_id,queue_wait_us,pure_gpu_us,end_to_end_us")


@pytest.mark.parametrize("path", ["tc2", "tc", "simt"])
def test_c4_sgemm_both_paths_within_tolerance(path):
    """All SGEMM kernels (3xTF32 tcgen05 on a CTA pair, the default; 3xTF32
    tcgen05 on one CTA; FP32 SIMT) against
    binary64 at 2048^2 and a non-multiple-of-128 size (SIMT fallback), in a
    fresh process since the path is chosen once per process (VGPU_SGEMM)."""
    import subprocess
    import sys
    code = r'''
import numpy as np
from paper_1511_07658_b200 import vgpu as V
for n in (2048, 200):
    rng = np.random.default_rng(7 + n)
    A = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    B = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    C = np.frombuffer(V.native_run_task(A.tobytes() + B.tobytes(), V.KernelDescriptor("sgemm")),
                      np.float32).reshape(n, n)
    rows = rng.choice(n, 48, replace=False)
    ref = A[rows].astype(np.float64) @ B.astype(np.float64)
    print(n, np.linalg.norm(C[rows] - ref) / np.linalg.norm(ref))
'''
    env = dict(os.environ, VGPU_SGEMM=path)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    for line in out.stdout.split("\n"):
        if line.strip():
            n, err = line.split()
            assert float(err) <= 1e-5, (path, n, err)


@pytest.mark.parametrize("sizes", [(512, 256, 768), (512, 384)])
def test_sgemm_mixed_sizes_in_one_batch(sizes):
    """One PS-1 batch of SGEMM jobs of different n through the GVM: every
    n % 256 == 0 takes the CTA-pair kernel (grid sized by the largest job,
    the smaller jobs' surplus pairs leave together), any n % 256 != 0 sends
    the batch to the 1-CTA tensor-core kernel. Full-matrix check against
    binary64 at the FP32 bar."""
    rng = np.random.default_rng(sum(sizes))
    mats = [(rng.uniform(-1, 1, (n, n)).astype(np.float32),
             rng.uniform(-1, 1, (n, n)).astype(np.float32)) for n in sizes]
    d, inst = _gvm(len(sizes), 8 * max(sizes) ** 2)
    with d:
        outs = [None] * len(sizes)

        def worker(i):
            h = V.req(inst)
            A, B = mats[i]
            outs[i] = h.run_task(A.tobytes() + B.tobytes(), V.KernelDescriptor("sgemm", 670, 344, 335))
            h.rls()
            h.close()

        ts = [threading.Thread(target=worker, args=(i,)) for i in range(len(sizes))]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    for (A, B), out, n in zip(mats, outs, sizes):
        C = np.frombuffer(out, np.float32).reshape(n, n)
        ref = A.astype(np.float64) @ B.astype(np.float64)
        err = np.linalg.norm(C - ref) / np.linalg.norm(ref)
        assert err <= 1e-5, (n, err)


@pytest.mark.parametrize("variant", [None, "11", "12"])
def test_ep_kernel_instances_match_their_oracle_order(variant):
    """The default EP instance (accepted pairs compacted per warp,
    range-specialised div/sqrt), the branch-free instance (VGPU_EP_VARIANT=11,
    lane-sequential sums) and compaction with the div/sqrt intrinsics (12)
    are each bit-exact
    against the oracle restating their reduction order, in a fresh process
    (the instance is chosen once per process)."""
    import subprocess
    import sys
    code = r'''
import os
from oracle import oracle
from paper_1511_07658_b200 import vgpu as V
lanes = os.environ.get("VGPU_EP_VARIANT") == "11"
for m, first, count in ((24, 0, 256), (28, 1536, 512), (20, 3, 5)):
    got = oracle.ep_from_bytes(V.native_run_task(oracle.ep_params_bytes(m, first, count),
                                                 V.KernelDescriptor("nas-ep")))
    want = oracle.ep_job(m, first, count, lanes=lanes)
    print(m, first, count, bytes(got) == bytes(want))
'''
    env = dict(os.environ)
    env.pop("VGPU_EP_VARIANT", None)
    if variant:
        env["VGPU_EP_VARIANT"] = variant
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l.split() for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 3 and all(l[-1] == "True" for l in lines), out.stdout


@pytest.mark.parametrize("mk", [8, 9, 10, 12, 20])
def test_ep_small_and_large_batches_bit_exact(mk):
    """EP batches of 2^mk pairs other than NPB's 2^16: 1, 2, 4 and 16 pairs
    per lane (the compaction kernel's remainder loop and ramp-up path) and
    4096 per lane, each bit-identical to the oracle."""
    m = mk + 6  # 64 batches
    ins = oracle.ep_params_bytes(m, 5, 40, mk=mk)
    got = oracle.ep_from_bytes(V.native_run_task(ins, V.KernelDescriptor("nas-ep")))
    want = oracle.ep_job(m, 5, 40, mk=mk)
    assert bytes(got) == bytes(want), (mk, got.sx, want.sx)
