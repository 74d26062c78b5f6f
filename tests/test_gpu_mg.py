"""[gpu] NAS MG (the paper's MG benchmark)
through the GVM, against the oracle (oracle/vgpu_oracle.c vo_mg_run, itself
pinned to NPB's published rnm2 for classes S, W, A, B in test_oracle.py).

Every grid operator evaluates mg.f's expression order with explicitly
rounded binary64 operations and the norm uses the shared fixed reduction
order, so rnm2 and rnmu must equal the oracle's BIT FOR BIT; NPB's own
verification (1e-8) must pass as well.
"""
import os
import struct
import threading

import pytest

from oracle import oracle
from paper_1511_07658_b200 import vgpu as V
from paper_1511_07658_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _bits(x: float) -> bytes:
    return struct.pack("<d", x)


def _run(inputs, shm):
    inst = f"mg{os.getpid()}_{len(inputs)}"
    V.unlink_os_instance(inst, len(inputs))
    cfg = V.GvmConfig(instance=inst, max_clients=len(inputs), barrier_size=len(inputs),
                      per_client_shm_bytes=shm, barrier_window=20000, clock=V.ClockMode.Real)
    d = V.GvmDaemon.start_os(cfg)
    outs, errs = [None] * len(inputs), []

    def worker(i):
        try:
            h = V.req(inst)
            outs[i] = h.run_task(inputs[i], V.KernelDescriptor("nas-mg", 5000, 30000, 5000, 64))
            h.rls()
            h.close()
        except Exception as e:  # pragma: no cover - reported below
            errs.append(repr(e))

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(len(inputs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    s = d.summary()
    d.stop()
    d.close()
    assert not errs, errs
    return outs, s


def _check(inp, out, cls):
    want = oracle.mg_run(inp)
    rnm2, rnmu, nx, nit = V.mg_result(out)
    assert _bits(rnm2) == _bits(want.rnm2), (cls, rnm2, want.rnm2)
    assert _bits(rnmu) == _bits(want.rnmu), (cls, rnmu, want.rnmu)
    assert (nx, nit) == (want.nx, want.nit)
    verify = V.mg_class(cls).rnm2_verify
    assert abs(rnm2 - verify) / verify <= 1e-8


def test_nas_mg_class_s_batch_of_8_bit_exact():
    """The paper's configuration: class S (32^3, 4 V-cycles), 8 SPMD
    processes in one batch (one launch: a thread-block cluster per job with
    comm3 / zero3 fused into the operators, mg_cluster_kernel)."""
    inp = V.mg_input_for_class("S")
    sz = W.Sizes()
    outs, s = _run([inp] * 8, W.region_bytes("mg", sz))
    assert s["device_tasks"] == 8
    for out in outs:
        _check(inp, out, "S")


def test_nas_mg_classes_w_and_a_bit_exact():
    inputs = [V.mg_input_for_class("W"), V.mg_input_for_class("A")]
    sz = W.Sizes()
    sz.mg_class = "A"
    outs, _ = _run(inputs, W.region_bytes("mg", sz))
    _check(inputs[0], outs[0], "W")
    _check(inputs[1], outs[1], "A")


def test_nas_mg_native_path_and_malformed_input():
    inp = V.mg_input_for_class("S")
    out = V.native_run_task(inp, V.KernelDescriptor("nas-mg", 5000, 30000, 5000, 64))
    _check(inp, out, "S")
    with pytest.raises(Exception):
        V.output_size("nas-mg", inp[:-8])


def test_nas_mg_class_s_both_device_paths_agree_bit_for_bit():
    """Class S through the launch-per-operator path (VGPU_MG_CLUSTER=0, a
    fresh process: the switch is read once) equals the oracle too, so both
    device schedules of mg.f give the same bits."""
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_1511_07658_b200 import vgpu as V\n"
            "inp = V.mg_input_for_class('S')\n"
            "out = V.native_run_task(inp, V.KernelDescriptor('nas-mg', 5000, 30000, 5000, 64))\n"
            "sys.stdout.write(out.hex())\n") % repo
    for flag in ("0", "1"):
        env = dict(os.environ, VGPU_MG_CLUSTER=flag)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        _check(V.mg_input_for_class("S"), bytes.fromhex(r.stdout.strip()), "S")
