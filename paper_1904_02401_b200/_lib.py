"""ctypes binding of the in-tree native library ``libalefsi_b200.so``.

This is the reference-side binding of the C ABI declared in
``include/alefsi_b200.h``.  The library must have been
built in-tree (``python -c "import __graft_entry__ as g; g.build()"``);
there is no fallback path — importing a device operation without the
library raises.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libalefsi_b200.so")

_i32, _i64, _f64, _p = C.c_int32, C.c_int64, C.c_double, C.c_void_p

# name -> argtypes (every function returns int status)
SIGNATURES = {
    "alefsi_abi_version": [],
    "alefsi_last_error": [],
    "alefsi_device_count": [_p],
    # host index structures
    "alefsi_pattern_build": [_i64, _i64, _p, _p, _p, _p],
    "alefsi_pattern_slots": [_i64, _p, _p, _i64, _i32, _p, _p],
    "alefsi_scatter_add_blocks": [_i64, _p, _p, _i64, _i32, _p, _i32, _p, _p, _i32],
    "alefsi_color_patches": [_i64, _p, _p, _p, _i64, _p, _p],
    "alefsi_pattern_match": [_i64, _p, _p, _p, _p, _p],
    "alefsi_split_extension": [_i64, _p, _p, _p, _p, _p, _p],
    # device multigrid hierarchy
    "alefsi_mg_create": [_i32, _i32, _i32, _i32, _f64, _p],
    "alefsi_mg_destroy": [_p],
    "alefsi_mg_set_stream": [_p, _p],
    "alefsi_mg_set_matrix": [_p, _i32, _i64, _i64, _p, _p, _p, _i64, _p, _p, _p],
    "alefsi_mg_set_patches": [_p, _i32, _i32, _p, _p, _p],
    "alefsi_mg_set_prolongation": [_p, _i32, _i64, _i64, _i64, _p, _p, _p],
    "alefsi_mg_set_constrained": [_p, _i32, _p],
    "alefsi_mg_factorize": [_p],
    "alefsi_mg_apply": [_p, _p, _p, _i32],
    "alefsi_mg_spmv": [_p, _i32, _p, _p, _p],
    "alefsi_mg_set_sell": [_p, _i32, _i32],
    "alefsi_mg_set_apply_split": [_p, _i32, _i32],
    "alefsi_mg_vanka_sweep": [_p, _i32, _p, _p],
    "alefsi_mg_restrict": [_p, _i32, _p, _p],
    "alefsi_mg_prolong_add": [_p, _i32, _p, _p],
    "alefsi_mg_coarse_solve": [_p, _p, _p],
    "alefsi_mg_get_inverses": [_p, _i32, _i32, _p],
    "alefsi_mg_info": [_p, _i32, _p],
    "alefsi_mg_use_graph": [_p, _i32],
    "alefsi_gmres": [_p, _p, _p, _f64, _f64, _i32, _i32, _p, _p, _p],
    "alefsi_gmres_workspace": [_p, _i32],
    "alefsi_kernel_stats": [_p, _p],
    "alefsi_mg_set_pattern": [_p, _i32, _i64, _i64, _p, _p, _i64, _p, _p],
    "alefsi_mg_asm_setup": [_p, _i32, _i32, _i64, _p, _p, _i32, _p, _p, _p, _i64, _p, _p, _p, _p],
    "alefsi_mg_asm_tables": [_p, _i32, _i32, _p, _p, _p],
    "alefsi_mg_asm_momentum": [_p, _i32, _p, _p, _p, _i64, _p, _p],
    "alefsi_mg_asm_outflow": [_p, _i32, _i64, _i32, _p, _p, _p, _p, _p, _p, _i64, _p, _p, _p],
    "alefsi_mg_asm_residual_tables": [_p, _i32, _p, _p, _p, _i64, _p, _p, _p],
    "alefsi_mg_get_matrix": [_p, _i32, _p, _p],
    "alefsi_mg_asm_residual": [_p, _i32, _p, _p, _p, _i32, _p],
    "alefsi_mg_profile": [_p, _i32],
    "alefsi_mg_profile_read": [_p, _p, _p, _i32],
}

_lib = None


class NativeError(RuntimeError):
    def __init__(self, code, message):
        super().__init__(f"[alefsi_b200 error {code}] {message}")
        self.code = code


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"native library {LIB_PATH} is missing; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    lib = C.CDLL(LIB_PATH)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name, None)
        if fn is None:
            continue            # reported by missing_symbols(); call() raises
        fn.argtypes = args
        fn.restype = C.c_char_p if name == "alefsi_last_error" else C.c_int
    _lib = lib
    return lib


def missing_symbols():
    lib = load()
    return [n for n in SIGNATURES if getattr(lib, n, None) is None]


def _conv(a):
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError("native call needs C-contiguous arrays")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):          # torch tensor (device or host)
        if not a.is_contiguous():
            raise ValueError("native call needs contiguous tensors")
        return a.data_ptr()
    return a


def call(name, *args):
    lib = load()
    fn = getattr(lib, name, None)
    if fn is None:
        raise NativeError(-1, f"symbol {name} missing from {LIB_PATH}")
    rc = fn(*[_conv(a) for a in args])
    if rc != 0:
        msg = lib.alefsi_last_error()
        raise NativeError(rc, msg.decode() if msg else "unknown error")
    return rc


def handle_ptr():
    return C.c_void_p()
