"""[gpu] Parity at BASELINE.json's PROCESS COUNTS, every job checked.

test_gpu_parity.py pins each kernel at its full problem size; here each
config runs exactly as bench.py runs it — all of its SPMD clients in ONE
GVM batch, so the batched task-table launches the bench times (BS: one
launch over 16 jobs, 32,768 CTAs; SGEMM: the CTA-pair grid (128, 1, 16);
the mixed batch: four kernel kinds at once) are the ones compared with the
oracle (oracle/oracle.py):

  C3  Black-Scholes 16 x 4 Mi options   every job, call and put halves:
                                        L1-relative <= 1e-6 vs binary64
  C4  SGEMM 16 x 2048^2                 every job, 64 sampled rows vs
                                        binary64: relative Frobenius <= 1e-5
  C5  16-process mixed batch            4 x vector-add bit-exact, 4 NAS EP
                                        quarter slices of class A bit-exact
                                        and their fold within 1e-8 of NPB,
                                        4 x Black-Scholes, 4 x SGEMM

Model: the reference's exact multi-process check (proj/tests/
acceptance.cpp:412-479, criterion 9: 8 processes, every result compared).
"""
import os
import threading

import numpy as np
import pytest

from oracle import oracle
from paper_1511_07658_b200 import vgpu as V

pytestmark = pytest.mark.gpu

BS_N = 4 << 20
MM_N = 2048
BS_DESC = V.KernelDescriptor("black-scholes", 1000, 13, 670)
MM_DESC = V.KernelDescriptor("sgemm", 670, 344, 335)


def _run_batch(jobs, shm):
    """All jobs as SPMD clients of one GVM whose barrier is the job count:
    one flush, one batch. Returns (outputs, batches)."""
    n = len(jobs)
    inst = f"cfg{os.getpid()}_{n}_{shm}"
    V.unlink_os_instance(inst, n)
    cfg = V.GvmConfig(instance=inst, max_clients=n, barrier_size=n, per_client_shm_bytes=shm,
                      barrier_window=10_000_000, clock=V.ClockMode.Real)
    outs = [None] * n
    errs = []
    with V.GvmDaemon.start_os(cfg) as gvm:
        def worker(i):
            try:
                h = V.req(inst)
                outs[i] = h.run_task(*jobs[i])
                h.rls()
                h.close()
            except Exception as e:  # pragma: no cover - reported below
                errs.append(repr(e))

        ts = [threading.Thread(target=worker, args=(i,)) for i in range(n)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        batches = gvm.batches()
    assert not errs, errs
    return outs, batches


def _bs_input(w):
    rng = np.random.default_rng(5347 + w)
    S = rng.uniform(5, 30, BS_N).astype(np.float32)
    X = rng.uniform(1, 100, BS_N).astype(np.float32)
    T = rng.uniform(0.25, 10, BS_N).astype(np.float32)
    return S, X, T


def _check_bs(inp, out):
    S, X, T = inp
    call, put = oracle.black_scholes(S, X, T)
    got = np.frombuffer(out, np.float32).astype(np.float64)
    assert got.size == 2 * BS_N
    for half, ref in ((got[:BS_N], call), (got[BS_N:], put)):
        l1 = np.sum(np.abs(half - ref)) / np.sum(np.abs(ref))
        assert l1 <= 1e-6, l1
        assert np.max(np.abs(half - ref)) < 5e-4


def _mm_input(w):
    rng = np.random.default_rng(1000 + w)
    return (rng.uniform(-1, 1, (MM_N, MM_N)).astype(np.float32),
            rng.uniform(-1, 1, (MM_N, MM_N)).astype(np.float32))


def _check_mm(inp, out, w):
    A, B = inp
    C = np.frombuffer(out, np.float32).reshape(MM_N, MM_N)
    rows = np.random.default_rng(w).choice(MM_N, 64, replace=False)
    ref = A[rows].astype(np.float64) @ B.astype(np.float64)
    err = np.linalg.norm(C[rows] - ref) / np.linalg.norm(ref)
    assert err <= 1e-5, (w, err)


def test_c3_black_scholes_16_processes_one_batch():
    ins = [_bs_input(w) for w in range(16)]
    jobs = [(S.tobytes() + X.tobytes() + T.tobytes(), BS_DESC) for S, X, T in ins]
    outs, batches = _run_batch(jobs, 12 * BS_N)
    assert [b["task_count"] for b in batches] == [16]
    for inp, out in zip(ins, outs):
        _check_bs(inp, out)


def test_c4_sgemm_16_processes_one_batch():
    ins = [_mm_input(w) for w in range(16)]
    jobs = [(A.tobytes() + B.tobytes(), MM_DESC) for A, B in ins]
    outs, batches = _run_batch(jobs, 8 * MM_N * MM_N)
    assert [b["task_count"] for b in batches] == [16]
    for w, (inp, out) in enumerate(zip(ins, outs)):
        _check_mm(inp, out, w)


def test_c5_mixed_16_processes_one_batch():
    """Worker w runs kind w % 4 (vecadd, EP, BS, SGEMM), the C5 mix of one
    GPU; the 4 EP workers split NAS EP class A into quarters."""
    n_va = 1 << 20
    jobs, want = [], []
    for w in range(16):
        kind = w % 4
        if kind == 0:
            rng = np.random.default_rng(41 + w)
            a = rng.uniform(-1000, 1000, n_va).astype(np.float32)
            b = rng.uniform(-1000, 1000, n_va).astype(np.float32)
            jobs.append((a.tobytes() + b.tobytes(), V.KernelDescriptor("vector-add", 168, 2, 84)))
            want.append(("va", oracle.vector_add(a, b).tobytes()))
        elif kind == 1:
            q = w // 4
            jobs.append((oracle.ep_params_bytes(28, 1024 * q, 1024),
                         V.KernelDescriptor("nas-ep", 1, 257, 1)))
            want.append(("ep", q))
        elif kind == 2:
            inp = _bs_input(w)
            jobs.append((b"".join(x.tobytes() for x in inp), BS_DESC))
            want.append(("bs", inp))
        else:
            inp = _mm_input(w)
            jobs.append((inp[0].tobytes() + inp[1].tobytes(), MM_DESC))
            want.append(("mm", inp))
    outs, batches = _run_batch(jobs, 12 * BS_N)
    assert [b["task_count"] for b in batches] == [16]
    parts = []
    for w, ((kind, ref), out) in enumerate(zip(want, outs)):
        if kind == "va":
            assert out == ref, w
        elif kind == "ep":
            got = oracle.ep_from_bytes(out)
            exp = oracle.ep_job(28, 1024 * ref, 1024)
            assert bytes(got) == bytes(exp), (w, got.sx, exp.sx)
            parts.append(got)
        elif kind == "bs":
            _check_bs(ref, out)
        else:
            _check_mm(ref, out, w)
    f = oracle.ep_fold(parts)
    assert f.pairs == 210832767
    sxv, syv = oracle.NPB_VERIFY[28]
    assert abs((f.sx - sxv) / sxv) < 1e-8 and abs((f.sy - syv) / syv) < 1e-8
