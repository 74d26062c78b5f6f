"""Python mirror of the reference's client/daemon API over the C-ABI.

Names, argument meanings and errors follow proj/include/vgpu/client.hpp and
daemon.hpp (the reference's C++ surface):

    daemon = GvmDaemon.start_os(GvmConfig(instance="gpu0", max_clients=4))
    h = req("gpu0")                       # VgpuHandle, $VGPU_INSTANCE fallback
    out = h.run_task(data, KernelDescriptor("vector-add", 60, 20, 40))
    h.rls(); daemon.stop()

NACK codes surface as VgpuError(code) exactly like the C++ VgpuError
(client.hpp:18-26); transport failures as TransportError. Every call goes
through libvgpu.so -> libvgpu_cuda.so; nothing here computes a payload.
"""
from __future__ import annotations

import ctypes as C
import enum
import struct
from dataclasses import dataclass, field
from typing import Optional, Sequence

from . import _native as N


class ErrCode(enum.IntEnum):  # proj/include/vgpu/message.hpp:42-51
    Phase = 1
    NoLease = 2
    Size = 3
    Pending = 4
    Payload = 5
    Full = 6
    Malformed = 7
    Internal = 8


class Phase(enum.IntEnum):  # proj/include/vgpu/daemon.hpp:36
    Idle = 0
    Leased = 1
    DataIn = 2
    Queued = 3
    Running = 4
    Done = 5
    Released = 6


class ClockMode(enum.IntEnum):
    Virtual = 0
    Real = 1


class DataPlane(enum.IntEnum):
    ZeroCopy = 0
    Snapshot = 1


class VgpuError(RuntimeError):
    def __init__(self, code: int, detail: str):
        super().__init__(detail)
        self.code = ErrCode(code) if 1 <= code <= 8 else code


class TransportError(RuntimeError):
    pass


class PayloadError(RuntimeError):
    pass


def _libs():
    return N.load()


def _check(rc: int) -> None:
    if rc == 0:
        return
    detail = (_libs().host.vgpu_last_error() or b"").decode(errors="replace")
    if 1 <= rc <= 8:
        raise VgpuError(rc, detail)
    if rc == 20:
        raise TransportError(detail)
    if rc == 21:
        raise ValueError(detail)
    if rc == 23:
        raise PayloadError(detail)
    raise RuntimeError(detail or f"vgpu error {rc}")


@dataclass
class KernelDescriptor:  # proj/include/vgpu/message.hpp:84-93
    payload_id: str = "identity"
    t_data_in: int = 0
    t_comp: int = 0
    t_data_out: int = 0
    grid_size: int = 1
    output_bytes: int = 0

    def to_c(self) -> N.DescriptorC:
        return N.DescriptorC(self.payload_id.encode(), self.t_data_in, self.t_comp,
                             self.t_data_out, self.grid_size, self.output_bytes)


@dataclass
class GvmConfig:  # proj/include/vgpu/daemon.hpp:21-33 (+ B200 fields)
    instance: str = "default"
    max_clients: int = 8
    per_client_shm_bytes: int = 1 << 20
    barrier_window: int = 2000
    barrier_size: int = 0
    t_init: int = 150000
    t_ctx_switch: int = 5000
    clock: ClockMode = ClockMode.Virtual
    scale: float = 1.0
    device_sms: int = 14
    device_max_kernels: int = 16
    device_slots_per_sm: int = 8
    cuda_device: int = 0
    data_plane: DataPlane = DataPlane.ZeroCopy
    _inst: bytes = field(default=b"", repr=False)

    def to_c(self) -> N.GvmConfigC:
        self._inst = self.instance.encode()
        return N.GvmConfigC(self._inst, self.max_clients, self.barrier_size,
                            self.per_client_shm_bytes, self.barrier_window, self.t_init,
                            self.t_ctx_switch, int(self.clock), self.cuda_device,
                            int(self.data_plane), self.device_sms, self.device_max_kernels,
                            self.device_slots_per_sm, self.scale)


class GvmDaemon:
    """One GVM: owns the CUDA context of `cuda_device` (daemon.hpp:69-96)."""

    def __init__(self, handle: int, cfg: GvmConfig):
        self._h = handle
        self.config = cfg

    @classmethod
    def start_os(cls, cfg: GvmConfig) -> "GvmDaemon":
        h = C.c_void_p()
        c = cfg.to_c()
        _check(_libs().host.vgpu_gvm_start_os(C.byref(c), C.byref(h)))
        return cls(h.value, cfg)

    def stop(self) -> None:
        if self._h:
            _check(_libs().host.vgpu_gvm_stop(self._h))

    def close(self) -> None:
        if self._h:
            _libs().host.vgpu_gvm_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def summary(self) -> dict:
        s = N.GvmSummary()
        _check(_libs().host.vgpu_gvm_summary_get(self._h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in N.GvmSummary._fields_}

    def tasks(self) -> list:
        n = C.c_uint32()
        _check(_libs().host.vgpu_gvm_tasks(self._h, None, 0, C.byref(n)))
        arr = (N.TaskMetricsC * max(1, n.value))()
        _check(_libs().host.vgpu_gvm_tasks(self._h, arr, n.value, C.byref(n)))
        return [{k: getattr(arr[i], k) for k, _ in N.TaskMetricsC._fields_ if k != "pad"}
                for i in range(n.value)]

    def batches(self) -> list:
        n = C.c_uint32()
        _check(_libs().host.vgpu_gvm_batches(self._h, None, 0, C.byref(n)))
        arr = (N.BatchMetricsC * max(1, n.value))()
        _check(_libs().host.vgpu_gvm_batches(self._h, arr, n.value, C.byref(n)))
        return [{k: getattr(arr[i], k) for k, _ in N.BatchMetricsC._fields_}
                for i in range(n.value)]

    def fold(self) -> list:
        """This GVM's partial record (GvmDaemon::fold_record, 16 doubles): the
        input of the single cross-GPU reduction."""
        out = (C.c_double * 16)()
        _check(_libs().host.vgpu_gvm_fold(self._h, out))
        return list(out)

    def metrics_csv(self) -> str:
        n = C.c_uint64()
        _check(_libs().host.vgpu_gvm_metrics_csv(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _check(_libs().host.vgpu_gvm_metrics_csv(self._h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def timeline_csv(self) -> str:
        """The measured schedule (CUDA events) in the reference's timeline
        schema: task_id,stream_id,kind,start_us,end_us."""
        n = C.c_uint64()
        _check(_libs().host.vgpu_gvm_timeline_csv(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _check(_libs().host.vgpu_gvm_timeline_csv(self._h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()


def rendezvous_publish(path: str, data: bytes) -> None:
    """Rank 0 publishes the NCCL unique id (atomic file rename)."""
    _check(_libs().host.vgpu_rendezvous_publish(path.encode(), data, len(data)))


def rendezvous_fetch(path: str, n: int, timeout_ms: int = 300000) -> bytes:
    """Ranks > 0 wait for the id rank 0 published."""
    buf = (C.c_uint8 * n)()
    _check(_libs().host.vgpu_rendezvous_fetch(path.encode(), buf, n, timeout_ms))
    return bytes(buf)


def fold_in_rank_order(flat, nranks: int) -> list:
    """The all-gathered records (rank-major) folded in rank order (C++)."""
    a = (C.c_double * (16 * nranks))(*flat)
    out = (C.c_double * 16)()
    _check(_libs().host.vgpu_fold_in_rank_order(a, nranks, out))
    return list(out)


def unlink_os_instance(instance: str, max_clients: int) -> None:
    _check(_libs().host.vgpu_unlink_instance(instance.encode(), max_clients))


def _as_buffer(data) -> tuple:
    mv = memoryview(data).cast("B")
    buf = (C.c_uint8 * len(mv)).from_buffer_copy(mv) if mv.readonly else \
        (C.c_uint8 * len(mv)).from_buffer(mv)
    return buf, len(mv)


class VgpuHandle:
    """The per-process virtual GPU (client.hpp:33-62)."""

    def __init__(self, handle: int):
        self._h = handle

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def close(self) -> None:
        if getattr(self, "_h", None):
            _libs().host.vgpu_client_free(self._h)
            self._h = None

    @property
    def client_id(self) -> int:
        return _libs().host.vgpu_client_id(self._h)

    @property
    def shm_bytes(self) -> int:
        return _libs().host.vgpu_client_shm_bytes(self._h)

    @property
    def phase(self) -> Phase:
        return Phase(_libs().host.vgpu_client_phase(self._h))

    def snd(self, data) -> None:
        buf, n = _as_buffer(data)
        _check(_libs().host.vgpu_client_snd(self._h, buf, n))

    def str(self, task: KernelDescriptor) -> None:
        d = task.to_c()
        _check(_libs().host.vgpu_client_str(self._h, C.byref(d)))

    def stp(self) -> bool:
        done = C.c_int()
        _check(_libs().host.vgpu_client_stp(self._h, C.byref(done)))
        return bool(done.value)

    def stp_wait(self) -> None:
        _check(_libs().host.vgpu_client_stp_wait(self._h))

    def rcv(self) -> bytes:
        cap = self.shm_bytes
        out = (C.c_uint8 * max(1, cap))()
        n = C.c_uint64()
        _check(_libs().host.vgpu_client_rcv(self._h, out, cap, C.byref(n)))
        return bytes(out[: n.value])

    def rls(self) -> None:
        _check(_libs().host.vgpu_client_rls(self._h))

    def run_task(self, data, task: KernelDescriptor) -> bytes:
        buf, n = _as_buffer(data)
        cap = self.shm_bytes
        out = (C.c_uint8 * max(1, cap))()
        got = C.c_uint64()
        d = task.to_c()
        _check(_libs().host.vgpu_client_run_task(self._h, buf, n, C.byref(d), out, cap,
                                                 C.byref(got)))
        return bytes(out[: got.value])

    # ---- in-place data plane (VgpuHandle::region / snd_region / rcv_region) ----

    def region(self) -> memoryview:
        """The leased region itself (page-locked by the GVM), writable."""
        base, n = C.c_void_p(), C.c_uint64()
        _check(_libs().host.vgpu_client_region(self._h, C.byref(base), C.byref(n)))
        return memoryview((C.c_uint8 * n.value).from_address(base.value)).cast("B")

    def snd_region(self, nbytes: int) -> None:
        _check(_libs().host.vgpu_client_snd_region(self._h, nbytes))

    def snd_region_at(self, offset: int, nbytes: int) -> None:
        """Input at [offset, offset + nbytes) of the region (results land at 0)."""
        _check(_libs().host.vgpu_client_snd_region_at(self._h, offset, nbytes))

    def rcv_region(self) -> memoryview:
        """The result in place (valid until the next SND or RLS)."""
        p, n = C.c_void_p(), C.c_uint64()
        _check(_libs().host.vgpu_client_rcv_region(self._h, C.byref(p), C.byref(n)))
        if n.value == 0:
            return memoryview(b"")
        return memoryview((C.c_uint8 * n.value).from_address(p.value)).cast("B").toreadonly()

    def run_task_region(self, nbytes: int, task: KernelDescriptor) -> memoryview:
        p, n = C.c_void_p(), C.c_uint64()
        d = task.to_c()
        _check(_libs().host.vgpu_client_run_task_region(self._h, nbytes, C.byref(d), C.byref(p),
                                                        C.byref(n)))
        if n.value == 0:
            return memoryview(b"")
        return memoryview((C.c_uint8 * n.value).from_address(p.value)).cast("B").toreadonly()


def req(instance: str = "") -> VgpuHandle:
    """Lease a VGPU (client.hpp:69; $VGPU_INSTANCE, else "default")."""
    h = C.c_void_p()
    _check(_libs().host.vgpu_client_req(instance.encode() if instance else None, C.byref(h)))
    return VgpuHandle(h.value)


def native_run_task(data, task: KernelDescriptor, cuda_device: int = 0,
                    out_cap: Optional[int] = None) -> bytes:
    """NativeVgpu::run_task: this process's own CUDA context (client.hpp:87-113)."""
    buf, n = _as_buffer(data)
    need = output_size(task.payload_id, data) if out_cap is None else out_cap
    out = (C.c_uint8 * max(1, need))()
    got = C.c_uint64()
    d = task.to_c()
    _check(_libs().host.vgpu_native_run_task(cuda_device, C.byref(d), buf, n, out, need,
                                             C.byref(got)))
    return bytes(out[: got.value])


# ---- device-level helpers (vgpu_cuda.h) ----------------------------------------

KERNELS = {"identity": 0, "vector-add": 1, "vector-scale": 2, "nas-ep": 3,
           "black-scholes": 4, "sgemm": 5, "vector-mul": 6, "nas-cg": 7,
           "electrostatics": 8, "nas-mg": 9}


def _cu_check(rc: int) -> None:
    if rc == 0:
        return
    lib = _libs().cuda
    detail = (lib.vgpu_cu_last_error() or b"").decode(errors="replace")
    name = (lib.vgpu_cu_strerror(rc) or b"").decode()
    if rc == 5:
        raise PayloadError(detail)
    raise RuntimeError(f"vgpu_cuda {name}: {detail}")


def output_size(payload_id: str, data) -> int:
    buf, n = _as_buffer(data)
    out = C.c_uint64()
    _cu_check(_libs().cuda.vgpu_cu_output_size(KERNELS[payload_id], buf, n, C.byref(out)))
    return out.value


def device_count() -> int:
    n = C.c_int()
    rc = _libs().cuda.vgpu_cu_device_count(C.byref(n))
    return n.value if rc == 0 else 0


def resident_bench(payload_id: str, inputs: Sequence[bytes], sets: int, warmup: int,
                   steps: int, device: int = 0, param: float = 2.0, pdl: bool = True,
                   main_only: bool = False) -> dict:
    """Device-only timing of the batched launch with inputs resident in HBM.
    main_only: SGEMM's tcgen05 GEMM alone (pre-pass outside the timed steps)."""
    bufs = [(C.c_uint8 * max(1, len(b))).from_buffer_copy(b if len(b) else b"\0")
            for b in inputs]
    ptrs = (C.c_void_p * len(bufs))(*[C.cast(b, C.c_void_p) for b in bufs])
    sizes = (C.c_uint64 * len(bufs))(*[len(b) for b in inputs])
    r = N.ResidentResult()
    _cu_check(_libs().cuda.vgpu_cu_resident_bench(device, KERNELS[payload_id], param,
                                                  len(bufs), ptrs, sizes, sets, warmup,
                                                  steps, (0 if pdl else 1) | (2 if main_only else 0),
                                                  C.byref(r)))
    return {k: getattr(r, k) for k, _ in N.ResidentResult._fields_}


def peak_probe(kind: str, device: int = 0) -> float:
    """Measured FMA pipe peak in TFLOP/s ("fp64" or "fp32") on `device`."""
    t = C.c_double()
    _cu_check(_libs().cuda.vgpu_cu_peak_probe(device, {"fp64": 0, "fp32": 1}[kind], C.byref(t)))
    return t.value


def link_probe(device: int = 0, nbytes: int = 256 << 20, reps: int = 8, shm: bool = False) -> dict:
    """Pinned host <-> HBM copy bandwidth (vgpu_cu_link_probe): H2D alone,
    D2H alone, both directions at once; GB/s (1e9 B/s). shm: POSIX shm pages
    registered in place (the data plane's memory) instead of cudaHostAlloc."""
    r = N.LinkResult()
    _cu_check(_libs().cuda.vgpu_cu_link_probe(device, nbytes, reps, 1 if shm else 0, C.byref(r)))
    return {"h2d_gbs": r.h2d_gbs, "d2h_gbs": r.d2h_gbs, "bidir_gbs": r.bidir_gbs,
            "bytes": r.bytes, "reps": reps, "host_memory": "shm, cudaHostRegister" if shm
            else "cudaHostAlloc"}


def model_simulate_fluid(style: int, n: int, t_in: int, t_comp: int, t_out: int, grid: int,
                         sms: int, ctas_per_sm: int, launch_us: int = 0, shared: bool = False) -> int:
    """simulate() with the B200 fluid block-scheduler spec (DeviceSpec::fluid_blocks: 1 queue
    order, 2 = shared when `shared`); launch_us = the fixed part of a kernel span
    (DeviceSpec::kernel_launch_us)."""
    return _libs().host.vgpu_model_simulate_fluid(style, n, t_in, t_comp, t_out, grid, sms,
                                                  ctas_per_sm, launch_us, 1 if shared else 0)


def launch_probe(device: int = 0) -> float:
    """The fixed part of an event-timed kernel span in us (vgpu_cu_launch_probe)."""
    t = C.c_double()
    _cu_check(_libs().cuda.vgpu_cu_launch_probe(device, C.byref(t)))
    return t.value


def task_shape(payload_id: str, data: bytes, device: int = 0) -> tuple:
    """(CTAs of one task, resident CTAs per SM) of the payload's kernel."""
    c, p = C.c_uint32(), C.c_uint32()
    buf = (C.c_uint8 * max(1, len(data))).from_buffer_copy(data) if data else None
    _cu_check(_libs().cuda.vgpu_cu_task_shape(device, KERNELS[payload_id], buf, len(data),
                                              C.byref(c), C.byref(p)))
    return c.value, p.value


def model_simulate(style: int, n: int, t_in: int, t_comp: int, t_out: int, grid: int = 1,
                   sms: int = 14, max_kernels: int = 16, slots: int = 8) -> int:
    return _libs().host.vgpu_model_simulate(style, n, t_in, t_comp, t_out, grid, sms,
                                            max_kernels, slots)


# ---- NPB CG problems (client side of the nas-cg payload) ----------------------

CG_HEADER = struct.Struct("<IIIId")   # vgpu_cg_header: n, nnz, niter, cgitmax, shift
CG_RESULT = struct.Struct("<ddIIQ")   # vgpu_cg_result: zeta, rnorm, niter, n, nnz


@dataclass
class CgClass:
    n: int
    nonzer: int
    niter: int
    shift: float
    zeta_verify: float


def cg_class(cls: str) -> CgClass:
    """NPB CG class parameters and the published zeta (S, W, A, B, C)."""
    n, nz, it = C.c_uint32(), C.c_uint32(), C.c_uint32()
    sh, zv = C.c_double(), C.c_double()
    _check(_libs().host.vgpu_cg_class(cls.encode()[:1], C.byref(n), C.byref(nz), C.byref(it),
                                      C.byref(sh), C.byref(zv)))
    return CgClass(n.value, nz.value, it.value, sh.value, zv.value)


def cg_make_input(n: int, nonzer: int, niter: int, shift: float) -> bytes:
    """The nas-cg input for an NPB-shaped problem (NPB makea, untimed in NPB)."""
    lib = _libs().host
    need = C.c_uint64()
    _check(lib.vgpu_cg_make_input(n, nonzer, niter, shift, None, 0, C.byref(need)))
    buf = (C.c_uint8 * need.value)()
    _check(lib.vgpu_cg_make_input(n, nonzer, niter, shift, buf, need.value, C.byref(need)))
    return bytes(buf)


def cg_input_for_class(cls: str, niter: Optional[int] = None) -> bytes:
    c = cg_class(cls)
    return cg_make_input(c.n, c.nonzer, c.niter if niter is None else niter, c.shift)


def cg_result(out: bytes) -> tuple:
    """(zeta, rnorm, niter, n, nnz) from a nas-cg result."""
    return CG_RESULT.unpack(bytes(out[:CG_RESULT.size]))


# ---- NPB MG problems (client side of the nas-mg payload) -------------------------

MG_RESULT = struct.Struct("<ddIIQ")  # vgpu_mg_result


@dataclass
class MgClass:
    nx: int
    nit: int
    coeffs: int
    rnm2_verify: float


def mg_class(cls: str) -> MgClass:
    """NPB MG class parameters and the published rnm2 (S, W, A, B, C)."""
    nx, nit, co, v = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_double()
    _check(_libs().host.vgpu_mg_class(cls.encode()[:1], C.byref(nx), C.byref(nit), C.byref(co),
                                      C.byref(v)))
    return MgClass(nx.value, nit.value, co.value, v.value)


def mg_make_input(nx: int, nit: int, coeffs: int) -> bytes:
    """The nas-mg input: header + NPB zran3's right-hand side (untimed in NPB)."""
    lib = _libs().host
    need = C.c_uint64()
    _check(lib.vgpu_mg_make_input(nx, nit, coeffs, None, 0, C.byref(need)))
    buf = (C.c_uint8 * need.value)()
    _check(lib.vgpu_mg_make_input(nx, nit, coeffs, buf, need.value, C.byref(need)))
    return bytes(buf)


def mg_input_for_class(cls: str, nit: Optional[int] = None) -> bytes:
    c = mg_class(cls)
    return mg_make_input(c.nx, c.nit if nit is None else nit, c.coeffs)


def mg_result(out: bytes) -> tuple:
    """(rnm2, rnmu, nx, nit) from a nas-mg result."""
    return MG_RESULT.unpack(bytes(out[:MG_RESULT.size]))[:4]


# ---- electrostatics inputs ------------------------------------------------------

ES_HEADER = struct.Struct("<IIIIfIII")  # vgpu_es_header


def es_input(atoms, nx: int, ny: int, nz: int, spacing: float) -> bytes:
    """electrostatics input: header + float32 atoms [natoms, 4] (x, y, z, q)."""
    import numpy as np
    a = np.ascontiguousarray(atoms, np.float32).reshape(-1, 4)
    return ES_HEADER.pack(a.shape[0], nx, ny, nz, spacing, 0, 0, 0) + a.tobytes()
