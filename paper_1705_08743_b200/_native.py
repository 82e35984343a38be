"""ctypes binding of the C ABI in include/semimat_b200.h.

The product path has exactly one backend: the sm_100a library built by
``_build.py``.  There is no CPU fallback -- if the library or a CUDA device is
missing, every matrix operation raises.
"""

from __future__ import annotations

import ctypes
from ctypes import c_int, c_longlong, c_size_t, c_void_p, POINTER

import torch

from . import _build

SMX_ANTI, SMX_DIST = 0, 1

_lib = None

# name -> (argtypes, restype)
_SIGS = {
    "smx_version": ([], c_int),
    "smx_error_string": ([c_int], ctypes.c_char_p),
    "smx_launch_count": ([], ctypes.c_ulonglong),
    "smx_set_bounded_fastpath": ([c_int], c_int),
    "smx_set_packed_tiles_per_cta": ([c_int], c_int),
    "smx_set_packed_producer_backoff": ([c_int], c_int),
    "smx_set_fw_lookahead": ([c_int], c_int),
    "smx_set_graphs": ([c_int], c_int),
    "smx_set_fw_side_lite": ([c_int], c_int),
    "smx_set_fw_split_3a": ([c_int], c_int),
    "smx_set_fw_pivot_pairs": ([c_int], c_int),
    "smx_set_fw_packed_panel": ([c_int], c_int),
    "smx_set_fw_panel_buffers": ([c_int], c_int),
    "smx_set_fw_pivot_blocked": ([c_int], c_int),
    "smx_set_bits_m4r": ([c_int], c_int),
    "smx_set_bool_persistent": ([c_int], c_int),
    "smx_set_bool_block": ([c_int], c_int),
    "smx_bool_persist_trace_arm": ([c_void_p, c_int], c_int),
    "smx_set_fw_block": ([c_int], c_int),
    "smx_set_fw_packed": ([c_int], c_int),
    "smx_fw_block_for": ([c_int, c_int], c_int),
    "smx_fw_trace_arm": ([c_int], c_int),
    "smx_fw_trace_read": ([c_void_p, c_void_p, c_int], c_int),
    "smx_fw_trace_offsets": ([c_void_p, c_void_p, c_int], c_int),
    "smx_semiring_gemm_u8": ([c_void_p] * 3 + [c_int] * 8 + [c_void_p], c_int),
    "smx_semiring_gemm_u16": ([c_void_p] * 3 + [c_int] * 8 + [c_void_p], c_int),
    "smx_semiring_gemm_u32": ([c_void_p] * 3 + [c_int] * 8 + [c_void_p], c_int),
    "smx_semiring_gemm_skip": ([c_void_p] * 3 + [c_int] * 10 + [c_void_p], c_int),
    "smx_semiring_gemm_skip_certified": ([c_void_p] * 3 + [c_int] * 10 + [c_void_p], c_int),
    "smx_fw_workspace_bytes": ([c_int, c_int, c_int], c_size_t),
    "smx_fw_u8": ([c_void_p, c_int, c_int, c_int, c_void_p, c_size_t, c_void_p], c_int),
    "smx_fw_u16": ([c_void_p, c_int, c_int, c_int, c_void_p, c_size_t, c_void_p], c_int),
    "smx_fw_u32": ([c_void_p, c_int, c_int, c_int, c_void_p, c_size_t, c_void_p], c_int),
    "smx_set_fw_host_stream": ([c_int], c_int),
    "smx_fw_host_workspace_bytes": ([c_int, c_int, c_int], c_size_t),
    "smx_fw_host_u8": ([c_void_p] * 3 + [c_int] * 3 + [c_void_p, c_size_t, c_void_p], c_int),
    "smx_fw_host_u16": ([c_void_p] * 3 + [c_int] * 3 + [c_void_p, c_size_t, c_void_p], c_int),
    "smx_fw_host_u32": ([c_void_p] * 3 + [c_int] * 3 + [c_void_p, c_size_t, c_void_p], c_int),
    "smx_fw_block": ([c_int], c_int),
    "smx_fw_pivot": ([c_void_p, c_int, c_int, c_int, c_int, c_void_p], c_int),
    "smx_bool_gemm_bits": ([c_void_p] * 3 + [c_int] * 7 + [c_void_p], c_int),
    "smx_bool_warshall_workspace_bytes": ([c_int, c_int], c_size_t),
    "smx_bool_warshall_bits": ([c_void_p, c_int, c_int, c_void_p, c_size_t, c_void_p], c_int),
    "smx_pack_bits": ([c_void_p, c_void_p] + [c_int] * 4 + [c_void_p], c_int),
    "smx_unpack_bits": ([c_void_p, c_void_p] + [c_int] * 4 + [c_void_p], c_int),
    "smx_transpose_u8": ([c_void_p, c_void_p] + [c_int] * 4 + [c_void_p], c_int),
    "smx_unpack_bits_transposed": ([c_void_p, c_void_p] + [c_int] * 4 + [c_void_p], c_int),
    "smx_from_edges": ([c_void_p, ctypes.c_longlong, c_void_p, c_int, c_int, c_int, c_int, c_void_p],
                       c_int),
    "smx_lane_entrywise":([c_void_p] * 3 + [c_int] * 6 + [c_void_p], c_int),
    "smx_bits_entrywise": ([c_void_p] * 3 + [c_int] * 4 + [c_void_p], c_int),
    "smx_int_issue_probe":([c_void_p, c_int, c_int, c_int, c_int, POINTER(c_longlong), c_void_p],
                            c_int),
}
_SIGS.update({
    "smx_bool_mul_tc_workspace_bytes": ([c_int, c_int, c_int], c_size_t),
    "smx_bool_mul_tc": ([c_void_p] * 3 + [c_int] * 6 + [c_void_p, c_size_t, c_void_p], c_int),
    "smx_bool_gemm_i8": ([c_void_p] * 4 + [c_int] * 7 + [c_void_p], c_int),
    "smx_bool_warshall_i8_workspace_bytes": ([c_int, c_int], c_size_t),
    "smx_bool_warshall_i8": ([c_void_p, c_int, c_int, c_void_p, c_size_t, c_void_p], c_int),
})
_SIGS.update({
    "smx_set_tc_tile_n": ([c_int], c_int),
    "smx_set_tc_pair": ([c_int], c_int),
    "smx_set_tc_batch_ks": ([c_int], c_int),
    "smx_set_tc_f4": ([c_int], c_int),
    "smx_set_tc_f4_batch_stages": ([c_int], c_int),
    "smx_bool_gemm_f4": ([c_void_p] * 3 + [c_int] * 7 + [c_void_p], c_int),
    "smx_bool_gemm_f4_batched": ([c_void_p] * 3 + [c_int] * 8 + [c_void_p], c_int),
    "smx_unpack_nibbles": ([c_void_p, c_void_p] + [c_int] * 4 + [c_void_p, c_void_p] + [c_int] * 4 + [c_void_p],
                           c_int),
    "smx_bool_mul_tc_batched_workspace_bytes": ([c_int, c_int, c_int, c_int], c_size_t),
    "smx_bool_mul_tc_batched": ([c_void_p, c_void_p, c_void_p] + [c_int] * 7 + [c_void_p, c_size_t, c_void_p],
                                c_int),
    "smx_bool_gemm_i8_batched": ([c_void_p, c_void_p, c_void_p] + [c_int] * 8 + [c_void_p], c_int),
    "smx_tc_trace_arm": ([c_void_p], c_int),
    "smx_lane_op": ([c_void_p] * 3 + [c_longlong, c_int, c_int, c_void_p], c_int),
    "smx_lanes_from_bits": ([c_void_p, c_int, c_void_p] + [c_int] * 4 + [c_void_p], c_int),
    "smx_lanes_to_bits": ([c_void_p, c_int, c_void_p] + [c_int] * 4 + [c_void_p], c_int),
    "smx_bool_mul_batched": ([c_void_p] * 3 + [c_int] * 7 + [c_longlong] * 3 + [c_void_p], c_int),
    "smx_bool_warshall_batched": ([c_void_p, c_int, c_int, c_int, c_longlong, c_void_p], c_int),
    "smx_fw_batched": ([c_void_p, c_int, c_int, c_int, c_longlong, c_int, c_int, c_void_p], c_int),
})
BCAST_FN = ctypes.CFUNCTYPE(c_int, c_void_p, c_size_t, c_int, c_void_p, c_void_p)
_SIGS.update({
    "smx_nccl_broadcast": ([c_void_p, c_size_t, c_int, c_void_p, c_void_p], c_int),
    "smx_nccl_async_error": ([c_void_p], c_int),
    "smx_copy_h2d": ([c_void_p, c_void_p, c_size_t, c_void_p], c_int),
    "smx_edges_first_invalid": ([c_void_p, c_longlong, c_int, c_longlong, c_void_p, c_void_p], c_int),
    "smx_fw_sharded_block": ([c_int, c_int, c_int], c_int),
    "smx_fw_sharded_workspace_bytes": ([c_int, c_int, c_int, c_int], c_size_t),
    "smx_fw_sharded": ([c_void_p] + [c_int] * 9 + [c_void_p, c_void_p, c_void_p, c_size_t, c_void_p], c_int),
    "smx_fw_sharded_u16": ([c_void_p] + [c_int] * 5 + [c_void_p, c_void_p, c_size_t, c_void_p], c_int),
})
_OPTIONAL: dict = {}


def declared_symbols() -> list[str]:
    return sorted(_SIGS) + sorted(_OPTIONAL)


def lib():
    """Load (building first if needed) the sm_100a library."""
    global _lib
    if _lib is None:
        path = _build.LIB
        if not path.exists():
            path = _build.build()
        handle = ctypes.CDLL(str(path))
        for name, (args, res) in list(_SIGS.items()) + list(_OPTIONAL.items()):
            fn = getattr(handle, name, None)
            if fn is None:
                if name in _SIGS:
                    raise RuntimeError(f"{path} does not export {name}")
                continue
            fn.argtypes = args
            fn.restype = res
        _lib = handle
    return _lib


def has(name: str) -> bool:
    return getattr(lib(), name, None) is not None


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().smx_error_string(rc).decode()
        raise RuntimeError(f"{what} failed: {msg} (code {rc})")


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("semimat_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    if dev.type != "cuda":
        raise RuntimeError(f"semimat_b200 tensors live on CUDA devices, got {dev}")
    return dev


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_ptr(device: torch.device | None = None) -> int:
    """cudaStream_t of torch's current stream on `device` (the raw accessor
    costs 0.1 us per call against 2 us for current_stream().cuda_stream)."""
    if _raw_stream is not None:
        idx = device.index if isinstance(device, torch.device) else device
        return _raw_stream(torch.cuda.current_device() if idx is None else idx)
    return torch.cuda.current_stream(device).cuda_stream


def workspace(nbytes: int, device: torch.device) -> torch.Tensor:
    """Scratch for one library call, from torch's stream-aware caching allocator."""
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


def ptr(t: torch.Tensor) -> int:
    return t.data_ptr()
