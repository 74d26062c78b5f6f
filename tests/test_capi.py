"""The C-ABI boundary (CPU): both libraries load, export every symbol their
headers declare, the codec/model entry points work, and device entry points
fail loudly (never fall back) when no GPU is present."""
import ctypes as C
import os
import re

import pytest

from paper_1511_07658_b200 import _native as N
from paper_1511_07658_b200 import vgpu as V

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    text = open(os.path.join(REPO, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    inline = set(re.findall(r"static\s+inline\s+[\w\s\*]+?\b(vgpu_[a-z0-9_]+)\s*\(", text))
    return sorted(set(re.findall(r"\b(vgpu_[a-z0-9_]+)\s*\(", text)) - inline)


@pytest.mark.parametrize("header,lib", [("vgpu_cuda.h", "cuda"), ("vgpu_c.h", "host")])
def test_every_declared_symbol_is_exported_and_bound(header, lib):
    libs = N.load()
    names = declared(header)
    assert len(names) > 10
    table = N.CUDA_API if lib == "cuda" else N.HOST_API
    for name in names:
        assert hasattr(getattr(libs, lib), name), name
        assert name in table, f"{name} not bound in _native"


def test_codec_through_the_c_abi():
    host = N.load().host
    out = (C.c_uint8 * 64)()
    n = C.c_uint64()
    assert host.vgpu_encode_frame(0x01, 7, 0, None, 0, out, 64, C.byref(n)) == 0
    assert n.value == 26
    assert bytes(out[:6]) == b"VGPU\x01\x01"
    op, cid, tid, plen = C.c_uint8(), C.c_uint32(), C.c_uint64(), C.c_uint64()
    assert host.vgpu_decode_frame(out, 26, C.byref(op), C.byref(cid), C.byref(tid), C.byref(plen)) == 0
    assert (op.value, cid.value, tid.value, plen.value) == (1, 7, 0, 0)
    out[0] = ord("X")
    assert host.vgpu_decode_frame(out, 26, None, None, None, None) == 1  # BadMagic
    assert host.vgpu_decode_frame(out, 10, None, None, None, None) == 4  # Truncated


def test_model_entry_points():
    assert V.model_simulate(0, 4, 20, 50, 20) == 210
    assert V.model_simulate(1, 4, 60, 20, 40) == 300
    host = N.load().host
    assert host.vgpu_model_no_vt(4, 100, 10, 20, 50, 20) == 790
    assert host.vgpu_model_classify(60, 20, 40) == 1  # IOIntensive


def test_payload_contracts_host_side():
    assert V.output_size("vector-add", b"\0" * 16) == 8
    assert V.output_size("black-scholes", b"\0" * 24) == 16
    assert V.output_size("sgemm", b"\0" * (8 * 9)) == 36
    with pytest.raises(V.PayloadError):
        V.output_size("vector-add", b"\0" * 3)
    with pytest.raises(V.PayloadError):
        V.output_size("sgemm", b"\0" * 24)


def test_no_silent_cpu_fallback_without_gpu(has_gpu):
    if has_gpu:
        pytest.skip("a GPU is present")
    assert V.device_count() == 0
    cfg = V.GvmConfig(instance=f"nogpu{os.getpid()}", max_clients=1)
    with pytest.raises(RuntimeError, match="CUDA"):
        V.GvmDaemon.start_os(cfg)
    with pytest.raises(RuntimeError):
        V.native_run_task(b"\0" * 16, V.KernelDescriptor("vector-add"))
