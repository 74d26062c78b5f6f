"""vgpu-b200: B200-native GPU Virtualization Manager (arXiv 1511.07658).

Many SPMD processes share one B200 through a GVM that owns the only CUDA
context; the reference's client API (VgpuHandle: REQ/SND/STR/STP/RCV/RLS)
is unchanged. The product is native code (libvgpu.so, libvgpu_cuda.so,
tools in bin/); this package is a thin ctypes layer over its C-ABI.
"""
from . import _native
from .vgpu import (ClockMode, DataPlane, ErrCode, GvmConfig, GvmDaemon, KernelDescriptor,
                   PayloadError, Phase, TransportError, VgpuError, VgpuHandle, device_count,
                   native_run_task, output_size, req, resident_bench, unlink_os_instance)

__all__ = ["ClockMode", "DataPlane", "ErrCode", "GvmConfig", "GvmDaemon", "KernelDescriptor",
           "PayloadError", "Phase", "TransportError", "VgpuError", "VgpuHandle", "device_count",
           "native_run_task", "output_size", "req", "resident_bench", "unlink_os_instance",
           "_native"]
