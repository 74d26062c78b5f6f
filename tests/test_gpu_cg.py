"""[gpu] The paper's remaining payloads: NAS CG and
VecMul through the GVM, against the oracle.

  nas-cg      NPB classes S, W, A in one batch: zeta within NPB's own
              verification epsilon (1e-10) of the published value and within
              1e-12 of the oracle; ||x - A z|| at rounding level; the result is
              bit-identical run to run (fixed reduction order)
  vector-mul  bit-exact vs the IEEE fp32 oracle, ragged sizes included
"""
import os
import threading

import numpy as np
import pytest

from oracle import oracle
from paper_1511_07658_b200 import vgpu as V

pytestmark = pytest.mark.gpu


def _gvm(n, shm, window=20000):
    inst = f"cg{os.getpid()}_{n}_{shm}"
    V.unlink_os_instance(inst, n)
    cfg = V.GvmConfig(instance=inst, max_clients=n, barrier_size=n, per_client_shm_bytes=shm,
                      barrier_window=window, clock=V.ClockMode.Real)
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


def test_nas_cg_classes_s_w_a_in_one_batch():
    classes = ["S", "W", "A", "S"]
    inputs = [V.cg_input_for_class(c) for c in classes]
    d, inst = _gvm(4, 24 << 20)
    with d:
        outs = _spmd(inst, inputs, V.KernelDescriptor("nas-cg", 50000, 1500000, 50000, 8))
        s = d.summary()
    assert s["device_tasks"] == 4
    for c, inp, out in zip(classes, inputs, outs):
        zeta, rnorm, niter, n, nnz = V.cg_result(out)
        want = V.cg_class(c)
        ref = oracle.cg_run(inp)
        assert abs(zeta - want.zeta_verify) / want.zeta_verify <= 1e-10, (c, zeta)
        assert abs(zeta - ref.zeta) / ref.zeta <= 1e-12, (c, zeta, ref.zeta)
        assert rnorm < 1e-12, (c, rnorm)
        assert (niter, n, nnz) == (want.niter, want.n, ref.nnz)
    # same input, same bits (cluster reductions in a fixed order)
    assert outs[0] == outs[3]


def test_nas_cg_native_path_and_generic_spd_matrix():
    # a non-NPB symmetric diagonally dominant matrix, few iterations, through
    # the per-process (non-virtualized) path
    rng = np.random.default_rng(7)
    n = 3000
    rows = [[] for _ in range(n)]
    for _ in range(6 * n):
        i, j = rng.integers(0, n, 2)
        v = rng.uniform(-1, 1)
        rows[i].append((j, v))
        rows[j].append((i, v))
    rowstr, col, val = [0], [], []
    for i in range(n):
        acc = {}
        for j, v in rows[i]:
            acc[j] = acc.get(j, 0.0) + v
        acc[i] = acc.get(i, 0.0) + 20.0
        for j in sorted(acc):
            col.append(j)
            val.append(acc[j])
        rowstr.append(len(col))
    nnz = len(col)
    hdr = V.CG_HEADER.pack(n, nnz, 3, 10, 5.0)
    body = np.array(rowstr, np.uint32).tobytes() + np.array(col, np.uint32).tobytes()
    pad = (-(len(hdr) + len(body))) % 8
    inp = hdr + body + b"\0" * pad + np.array(val, np.float64).tobytes()
    assert V.output_size("nas-cg", inp) == V.CG_RESULT.size
    out = V.native_run_task(inp, V.KernelDescriptor("nas-cg"))
    zeta, rnorm, niter, nn, nz = V.cg_result(out)
    ref = oracle.cg_run(inp)
    assert (niter, nn, nz) == (3, n, nnz)
    assert abs(zeta - ref.zeta) / abs(ref.zeta) <= 1e-12, (zeta, ref.zeta)
    assert abs(rnorm - ref.rnorm) <= 1e-9 * max(1.0, ref.rnorm), (rnorm, ref.rnorm)


def test_nas_cg_malformed_input_is_a_payload_error():
    inp = V.cg_input_for_class("S")
    d, inst = _gvm(1, 2 << 20)
    with d:
        h = V.req(inst)
        h.snd(inp[:-8])
        with pytest.raises(V.VgpuError) as e:
            h.str(V.KernelDescriptor("nas-cg"))
            h.stp_wait()
        assert e.value.code == V.ErrCode.Payload
        h.close()


@pytest.mark.parametrize("n", [1 << 20, 1000003, 4, 1])
def test_vector_mul_bit_exact(n):
    rng = np.random.default_rng(n)
    ins, want = [], []
    for _ in range(4):
        a = rng.uniform(-1000, 1000, n).astype(np.float32)
        b = rng.uniform(-1000, 1000, n).astype(np.float32)
        ins.append(a.tobytes() + b.tobytes())
        want.append(oracle.vector_mul(a, b).tobytes())
    d, inst = _gvm(4, max(8 * n, 4096))
    with d:
        outs = _spmd(inst, ins, V.KernelDescriptor("vector-mul", 168, 2, 84))
    assert outs == want


@pytest.mark.parametrize("mode", ["0", "1", "2", "grid"])
def test_nas_cg_every_vector_placement(mode):
    """Each placement of the CG vectors (cluster kernel, the default, with
    VGPU_CG_MODE: 0 HBM, 1 p staged in shared memory, 2 everything in shared
    memory with DSMEM pushes; and the opt-in grid kernel, VGPU_CG_GRID=1:
    plain co-resident CTAs with a global-memory barrier) meets NPB's verification
    and the oracle, in a fresh process (the switches are read once per
    process). Classes S and W in one batch, and a class S alone."""
    import subprocess
    import sys
    code = r'''
import threading
from oracle import oracle
from paper_1511_07658_b200 import vgpu as V
for classes in (["S", "W"], ["S"]):
    ins = [V.cg_input_for_class(c) for c in classes]
    outs = [V.native_run_task(i, V.KernelDescriptor("nas-cg")) for i in ins] if len(classes) == 1 else None
    if outs is None:
        inst = "cgm%d" % len(classes)
        V.unlink_os_instance(inst, len(classes))
        cfg = V.GvmConfig(instance=inst, max_clients=len(classes), barrier_size=len(classes),
                          per_client_shm_bytes=8 << 20, barrier_window=20000, clock=V.ClockMode.Real)
        outs = [None] * len(classes)
        with V.GvmDaemon.start_os(cfg):
            def w(k):
                h = V.req(inst)
                outs[k] = h.run_task(ins[k], V.KernelDescriptor("nas-cg"))
                h.rls(); h.close()
            ts = [threading.Thread(target=w, args=(k,)) for k in range(len(classes))]
            [t.start() for t in ts]; [t.join() for t in ts]
    for c, i, o in zip(classes, ins, outs):
        zeta = V.cg_result(o)[0]
        ref = oracle.cg_run(i).zeta
        want = V.cg_class(c).zeta_verify
        print(c, abs(zeta - want) / want <= 1e-10 and abs(zeta - ref) / ref <= 1e-12)
'''
    env = dict(os.environ, VGPU_CG_GRID="1") if mode == "grid" else \
        dict(os.environ, VGPU_CG_MODE=mode)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l.split() for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 3 and all(l[-1] == "True" for l in lines), out.stdout


def _es_atoms(seed, natoms, nx, ny, nz, h):
    rng = np.random.default_rng(seed)
    at = np.empty((natoms, 4), np.float32)
    at[:, 0] = rng.uniform(0, nx * h, natoms)
    at[:, 1] = rng.uniform(0, ny * h, natoms)
    at[:, 2] = rng.uniform(0, nz * h, natoms)
    at[:, 3] = rng.uniform(-1, 1, natoms)
    return at


def test_electrostatics_ragged_lattices_vs_binary64_oracle():
    """Direct Coulomb summation (the paper's ES) on lattices that do not
    divide the CTA tile (x: 64 points, y: 8 rows), three clients in one batch:
    L1-relative <= 1e-5 against the binary64 oracle (FP32 terms through
    MUFU rsqrt.approx, ~2^-22 each; a single lattice point with 513 mixed
    charges measured 1.5e-6)."""
    shapes = [(2000, 70, 33, 5, 0.5), (513, 1, 1, 1, 0.25), (4096, 64, 64, 3, 0.3)]
    ins = [V.es_input(_es_atoms(i, *s), *s[1:]) for i, s in enumerate(shapes)]
    d, inst = _gvm(3, max(len(b) for b in ins) + (1 << 16))
    with d:
        outs = _spmd(inst, ins, V.KernelDescriptor("electrostatics", 20, 30000, 20, 288))
    for s, inp, out in zip(shapes, ins, outs):
        got = np.frombuffer(out, np.float32).reshape(s[3], s[2], s[1]).astype(np.float64)
        ref = oracle.es(inp)
        err = np.abs(got - ref).sum() / np.abs(ref).sum()
        assert err <= 1e-5, (s, err)


def test_electrostatics_paper_size_100k_atoms():
    """The paper's ES size: 100K atoms, 25 lattice slices (64 x 64 each)."""
    at = _es_atoms(11, 100000, 64, 64, 25, 0.5)
    inp = V.es_input(at, 64, 64, 25, 0.5)
    out = V.native_run_task(inp, V.KernelDescriptor("electrostatics"))
    got = np.frombuffer(out, np.float32).reshape(25, 64, 64).astype(np.float64)
    ref = oracle.es(inp)
    err = np.abs(got - ref).sum() / np.abs(ref).sum()
    assert err <= 1e-5, err
    with pytest.raises(Exception):
        V.native_run_task(inp[:-4], V.KernelDescriptor("electrostatics"))


def test_nas_cg_malformed_interior_rowstr_stays_in_bounds():
    """Only rowstr's ends are validated on the host; interior entries beyond
    nnz and column indices beyond n are clamped in the kernel, so a bad
    client gets a (meaningless) result instead of a device fault that would
    take the shared GVM context down. The next job still verifies."""
    good = V.cg_input_for_class("S", niter=1)
    n, nnz = V.CG_HEADER.unpack(good[:24])[:2]
    bad = bytearray(good)
    rs = np.frombuffer(bad, np.uint32, n + 1, 24)
    rs[n // 2] = 0xFFFFFFF0
    col = np.frombuffer(bad, np.uint32, nnz, 24 + 4 * (n + 1))
    col[:100] = 0xFFFFFFFF
    V.native_run_task(bytes(bad), V.KernelDescriptor("nas-cg"))
    out = V.native_run_task(V.cg_input_for_class("S"), V.KernelDescriptor("nas-cg"))
    zeta = V.cg_result(out)[0]
    assert abs(zeta - V.cg_class("S").zeta_verify) / V.cg_class("S").zeta_verify <= 1e-10


@pytest.mark.parametrize("style", ["ps1", "ps2"])
def test_every_payload_kind_in_one_gvm_batch(style):
    """Seven clients, seven payload kinds (vector-add, vector-mul, nas-ep,
    black-scholes, sgemm, nas-cg, electrostatics) in one barrier batch: the
    PS-1 launch grouping (one launch per kind, compute-intensive descriptors)
    and PS-2 (per-stream triples, I/O-intensive descriptors) both give every
    client its own oracle answer."""
    rng = np.random.default_rng(21)
    n = 4099
    a = rng.uniform(-10, 10, n).astype(np.float32)
    b = rng.uniform(-10, 10, n).astype(np.float32)
    S = rng.uniform(5, 30, 1000).astype(np.float32)
    X = rng.uniform(1, 100, 1000).astype(np.float32)
    T = rng.uniform(0.25, 10, 1000).astype(np.float32)
    A = rng.uniform(-1, 1, (128, 128)).astype(np.float32)
    B = rng.uniform(-1, 1, (128, 128)).astype(np.float32)
    cg = V.cg_input_for_class("S", niter=2)
    es = V.es_input(_es_atoms(4, 700, 20, 9, 3, 0.5), 20, 9, 3, 0.5)
    jobs = [("vector-add", a.tobytes() + b.tobytes()), ("vector-mul", a.tobytes() + b.tobytes()),
            ("nas-ep", oracle.ep_params_bytes(20, 1, 6)),
            ("black-scholes", S.tobytes() + X.tobytes() + T.tobytes()),
            ("sgemm", A.tobytes() + B.tobytes()), ("nas-cg", cg), ("electrostatics", es)]
    # the reference's batch_style: PS-1 for a compute-intensive majority,
    # PS-2 for an I/O-intensive one (proj/src/model.cpp:38-41)
    t = (10, 500000, 10) if style == "ps1" else (5000, 10, 5000)
    # a long barrier window: the batch flushes when all seven have arrived
    d, inst = _gvm(len(jobs), max(len(j[1]) for j in jobs) + (1 << 16), window=10_000_000)
    outs = [None] * len(jobs)
    errs = []

    def worker(i):
        try:
            h = V.req(inst)
            outs[i] = h.run_task(jobs[i][1], V.KernelDescriptor(jobs[i][0], *t))
            h.rls()
            h.close()
        except Exception as e:  # pragma: no cover
            errs.append(repr(e))

    with d:
        ts = [threading.Thread(target=worker, args=(i,)) for i in range(len(jobs))]
        [x.start() for x in ts]
        [x.join() for x in ts]
        batches = d.batches()
    assert not errs, errs
    assert batches and all(bt["task_count"] == len(jobs) for bt in batches), batches
    assert {bt["style"] for bt in batches} == {0 if style == "ps1" else 1}, batches
    assert outs[0] == oracle.vector_add(a, b).tobytes()
    assert outs[1] == oracle.vector_mul(a, b).tobytes()
    assert bytes(oracle.ep_from_bytes(outs[2])) == bytes(oracle.ep_job(20, 1, 6))
    call, put = oracle.black_scholes(S, X, T)
    got = np.frombuffer(outs[3], np.float32)
    assert np.abs(got[:1000] - call).sum() / np.abs(call).sum() <= 1e-6
    C = np.frombuffer(outs[4], np.float32).reshape(128, 128)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    assert np.linalg.norm(C - ref) / np.linalg.norm(ref) <= 1e-5
    zeta = V.cg_result(outs[5])[0]
    assert abs(zeta - oracle.cg_run(cg).zeta) / abs(oracle.cg_run(cg).zeta) <= 1e-12
    vg = np.frombuffer(outs[6], np.float32).astype(np.float64)
    ve = oracle.es(es).ravel()
    assert np.abs(vg - ve).sum() / np.abs(ve).sum() <= 1e-5


@pytest.mark.parametrize("switch", ["auto", "groups2", "groups3", "solo", "off"])
def test_nas_cg_group_mode_class_a(switch):
    """Group mode (k_cg.cuh): a job over several clusters that exchange dot
    partials and p / z slices through the workspace. Eight class-A jobs in
    one GVM batch and one class-A job on the native path, each meeting
    NPB's verification (1e-10) and the oracle (1e-12), the eight batch
    results bit-identical (same input, same fixed reduction order; not under
    solo, where arrival order picks each job's split). auto:
    the host's shape (group mode for the single native job only);
    groups2/3: VGPU_CG_GROUPS forces 2 / 3 clusters per job in the batch
    too; solo: forced 2 with VGPU_CG_JOIN_US=0, so the first cluster of a
    job usually claims it alone and its siblings exit (the fallback for
    clusters that are not co-resident); off: VGPU_CG_GROUPS=1."""
    import subprocess
    import sys
    code = r'''
import threading
from oracle import oracle
from paper_1511_07658_b200 import vgpu as V
inp = V.cg_input_for_class("A")
want = V.cg_class("A").zeta_verify
ref = oracle.cg_run(inp).zeta
inst = "cgg8"
V.unlink_os_instance(inst, 8)
cfg = V.GvmConfig(instance=inst, max_clients=8, barrier_size=8, per_client_shm_bytes=len(inp) + (1 << 16),
                  barrier_window=200000, clock=V.ClockMode.Real)
outs = [None] * 8
with V.GvmDaemon.start_os(cfg):
    def w(k):
        h = V.req(inst)
        outs[k] = h.run_task(inp, V.KernelDescriptor("nas-cg"))
        h.rls(); h.close()
    ts = [threading.Thread(target=w, args=(k,)) for k in range(8)]
    [t.start() for t in ts]; [t.join() for t in ts]
outs.append(V.native_run_task(inp, V.KernelDescriptor("nas-cg")))
for o in outs:
    zeta = V.cg_result(o)[0]
    print("job", abs(zeta - want) / want <= 1e-10 and abs(zeta - ref) / ref <= 1e-12, zeta)
print("same", all(o == outs[0] for o in outs[:8]))
'''
    env = dict(os.environ, VGPU_CG_VERBOSE="1")
    if switch == "solo":
        env["VGPU_CG_JOIN_US"] = "0"
        env["VGPU_CG_GROUPS"] = "2"
    elif switch.startswith("groups"):
        env["VGPU_CG_GROUPS"] = switch[-1]
    elif switch == "off":
        env["VGPU_CG_GROUPS"] = "1"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l.split() for l in out.stdout.splitlines() if l.strip()]
    jobs = [l for l in lines if l[0] == "job"]
    assert len(jobs) == 9 and all(l[1] == "True" for l in jobs), out.stdout
    if switch != "solo":  # solo: each job grouped or alone by arrival order, so its sum order varies
        assert ["same", "True"] in lines, out.stdout
    if switch == "off":
        assert "groups=1" in out.stderr and "groups=2" not in out.stderr, out.stderr[-2000:]
    else:
        import re
        shapes = {(int(j), int(g)) for j, g in re.findall(r"jobs=(\d+) width=\d+ groups=(\d+)", out.stderr)}
        if switch == "auto":  # the batch keeps one cluster per job, the single job is grouped
            assert (8, 1) in shapes and any(j == 1 and g > 1 for j, g in shapes), shapes
        else:
            assert (8, int(switch[-1]) if switch != "solo" else 2) in shapes, shapes
