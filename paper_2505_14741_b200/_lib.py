"""ctypes binding of the in-tree C-ABI library (include/parastep_b200.h).

The library is the product: there is no CPU fallback. Importing a module that
needs it raises ``NativeLibraryError`` when the .so is missing or when no CUDA
device is present, naming what is wrong.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libparastep_b200.so")

PS_F64, PS_F32, PS_BF16 = 0, 1, 2
PS_MAX_CYCLE = 16
PS_EINVAL, PS_ECUDA, PS_EUNSUP = 1001, 1002, 1003


class NativeLibraryError(RuntimeError):
    """The CUDA extension is missing or failed; the product path never falls back."""


class ps_step(C.Structure):
    _fields_ = [("c", C.c_double), ("sqrt_a", C.c_double), ("sigma", C.c_double),
                ("t", C.c_int32), ("noisy", C.c_int32)]


class ps_mlp(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("activation", C.c_int32), ("data_dim", C.c_int32),
                ("embed_dim", C.c_int32), ("dims", C.c_int32 * 17),
                ("W", C.c_void_p * 16), ("b", C.c_void_p * 16), ("temb_table", C.c_void_p)]


class ps_dit_config(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "channels", "frames", "height", "width", "layout", "patch", "hidden", "depth", "heads",
        "mlp_hidden", "freq_dim", "max_batch", "precision", "gemm_impl", "text_tokens",
        "rope")]


class ps_dit_weights(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("W", C.POINTER(C.c_void_p)),
                ("b", C.POINTER(C.c_void_p)), ("pos", C.c_void_p), ("freq_table", C.c_void_p),
                ("freq_rows", C.c_int32), ("text", C.c_void_p), ("rope", C.c_void_p)]


class ps_unet_op(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "kind", "layer", "pre", "in1", "in2", "c1", "c2", "h", "w", "taps", "resample", "cout",
        "temb_layer", "temb_off", "resid", "out", "out_bf16", "act", "heads")] + [
        ("eps", C.c_float), ("out2", C.c_int32)]


class ps_unet_config(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "in_channels", "height", "width", "groups", "freq_dim", "temb_dim", "temb_cols",
        "max_batch", "n_ops", "n_bufs")] + [("ops", C.POINTER(ps_unet_op)),
                                            ("bufs", C.POINTER(C.c_void_p))]


_SIGS = {
    "ps_last_error": (C.c_char_p, []),
    "ps_version": (C.c_int, []),
    "ps_sm_count": (C.c_int, [C.c_int]),
    "ps_rng_normal": (C.c_int, [C.c_void_p, C.c_int64, C.c_uint64, C.c_uint64, C.c_uint64,
                                C.c_int, C.c_void_p]),
    "ps_rng_normal_dev": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_uint64, C.c_uint64,
                                    C.c_int, C.c_void_p]),
    "ps_rng_uniform": (C.c_int, [C.c_void_p, C.c_int64, C.c_uint64, C.c_uint64, C.c_uint64,
                                 C.c_int, C.c_void_p]),
    "ps_rng_xavier": (C.c_int, [C.c_void_p, C.c_int64, C.c_uint64, C.c_uint64, C.c_double,
                                C.c_int, C.c_void_p]),
    "ps_sched_cycle": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_void_p,
                                 C.c_int, C.POINTER(ps_step), C.POINTER(C.c_void_p),
                                 C.POINTER(C.c_void_p), C.c_int, C.c_int, C.POINTER(ps_step),
                                 C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_void_p]),
    "ps_sched_step_z": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                  C.c_int, C.POINTER(ps_step), C.c_void_p]),
    "ps_mlp_workspace_bytes": (C.c_size_t, [C.POINTER(ps_mlp), C.c_int]),
    "ps_mlp_forward": (C.c_int, [C.POINTER(ps_mlp), C.c_void_p, C.POINTER(C.c_int32), C.c_int,
                                 C.c_void_p, C.c_void_p, C.c_void_p]),
    "ps_dit_create": (C.c_int, [C.POINTER(ps_dit_config), C.POINTER(ps_dit_weights),
                                C.POINTER(C.c_void_p)]),
    "ps_dit_forward": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_int32), C.c_int,
                                 C.c_void_p, C.c_void_p]),
    "ps_dit_destroy": (C.c_int, [C.c_void_p]),
    "ps_dit_condition_reserve": (C.c_int, [C.c_void_p, C.c_int]),
    "ps_dit_condition": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "ps_dit_condition_clear": (C.c_int, [C.c_void_p]),
    "ps_dit_condition_chunk": (C.c_int, [C.c_void_p]),
    "ps_dit_flops": (C.c_double, [C.c_void_p]),
    "ps_dit_kernels_per_forward": (C.c_int, [C.c_void_p]),
    "ps_dit_bench_gemm": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]),
    "ps_gemm_stamps": (C.c_int, [C.POINTER(C.c_longlong)]),
    "ps_gemm_tune": (C.c_int, [C.c_int]),
    "ps_gemm_force": (None, [C.c_int, C.c_int]),
    "ps_gemm_probe": (C.c_float, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]),
    "ps_unet_create": (C.c_int, [C.POINTER(ps_unet_config), C.POINTER(ps_dit_weights),
                                 C.POINTER(C.c_void_p)]),
    "ps_unet_forward": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_int32), C.c_int,
                                  C.c_void_p, C.c_void_p]),
    "ps_unet_destroy": (C.c_int, [C.c_void_p]),
    "ps_unet_kernels_per_forward": (C.c_int, [C.c_void_p]),
    "ps_dev_alloc": (C.c_int, [C.c_size_t, C.POINTER(C.c_void_p)]),
    "ps_dev_free": (C.c_int, [C.c_void_p]),
    "ps_ipc_get_handle": (C.c_int, [C.c_void_p, C.c_void_p]),
    "ps_ipc_open_handle": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "ps_ipc_close": (C.c_int, [C.c_void_p]),
    "ps_peer_signal": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64, C.c_void_p]),
    "ps_peer_wait": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64, C.c_void_p]),
    "ps_peer_epoch_advance": (C.c_int, [C.c_void_p, C.c_void_p]),
    "ps_copy": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "ps_stamp": (C.c_int, [C.c_void_p, C.c_void_p]),
    "ps_traj_pack_bytes": (C.c_int64, [C.c_int, C.c_int64]),
    "ps_traj_pack": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.c_int, C.c_int64, C.c_int, C.c_void_p, C.c_void_p]),
    "ps_traj_diff": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                               C.c_int64, C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
    "ps_attn_test": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                               C.c_int, C.c_void_p]),
    "ps_attn_probe": (C.c_float, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]),
    "ps_fmha_set_poly": (C.c_int, [C.c_int]),
    "ps_gemm_test": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                               C.c_int, C.c_int, C.c_int, C.c_void_p]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load(require_gpu: bool = False) -> C.CDLL:
    """Load (once) and type the library; optionally insist on a CUDA device."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "or `make -C paper_2505_14741_b200/csrc`")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    if require_gpu:
        import torch

        if not torch.cuda.is_available():
            raise NativeLibraryError("no CUDA device: the ParaStep B200 path has no CPU fallback")
    return _lib


def check(rc: int, what: str) -> None:
    """Map a C-ABI status to the reference's exception types."""
    if rc == 0:
        return
    msg = (_lib.ps_last_error() or b"").decode()
    if rc == PS_EINVAL:
        from .errors import DimensionError
        raise DimensionError(f"{what}: {msg}")
    raise NativeLibraryError(f"{what} failed (code {rc}): {msg}")


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t) -> int:
    return int(t.data_ptr()) if t is not None else 0


def ptr_array(ptrs) -> "C.Array":
    arr = (C.c_void_p * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr


def step_array(steps) -> "C.Array":
    arr = (ps_step * max(1, len(steps)))()
    for i, s in enumerate(steps):
        arr[i] = s
    return arr
