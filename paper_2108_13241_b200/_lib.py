"""ctypes binding of liblbm19.so (include/lbm19.h).

The shared library is built in-tree (`python -m paper_2108_13241_b200.build`
or `__graft_entry__.build()`).  There is no CPU fallback: if the library is
missing or no CUDA device is present, every solver entry point raises.
"""

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# LBM_LIB: an alternative build of the same ABI (the experiments library,
# python -m paper_2108_13241_b200.build --experiments -> exp_lib/liblbm19_exp.so)
LIB_PATH = os.environ.get("LBM_LIB") or os.path.join(_HERE, "_lib", "liblbm19.so")

LBM_OK, LBM_EINVAL, LBM_ESTATE, LBM_ENOMEM, LBM_ECUDA, LBM_ENCCL, LBM_EDIVERGED = \
    0, -1, -2, -3, -4, -5, -6
LBM_F32, LBM_F64 = 0, 1
LAYOUT_CODES = {"dense": 0, "tile": 1, "bitmask_node": 2, "pointer_tile": 3}
SCHEME_CODES = {"ab": 0, "aa": 1}
ABI_VERSION = 2
HALO_BLOB_BYTES = 512


class LbmDesc(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
                ("nz_global", C.c_int32), ("z0", C.c_int32),
                ("periodic", C.c_int32 * 3), ("dtype", C.c_int32),
                ("layout", C.c_int32), ("tile", C.c_int32 * 3),
                ("device", C.c_int32), ("omega", C.c_double), ("scheme", C.c_int32)]


class LbmStats(C.Structure):
    _fields_ = [("n_nodes", C.c_int64), ("n_nonsolid", C.c_int64),
                ("visits_per_step", C.c_int64), ("n_slots", C.c_int64),
                ("plane_stride", C.c_int64), ("n_tiles", C.c_int64),
                ("step_count", C.c_int64), ("visited_nodes_total", C.c_int64),
                ("device_bytes", C.c_int64), ("launches_total", C.c_int64),
                ("last_step_ms", C.c_double), ("meta_bytes_per_step", C.c_int64),
                ("parity", C.c_int32),
                ("initialized", C.c_int32), ("scheme", C.c_int32), ("tile_work_list", C.c_int32)]


P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
D = C.c_double
PD = C.POINTER(C.c_double)

# (name, restype, argtypes) for every symbol of include/lbm19.h
SIGNATURES = [
    ("lbm_last_error", C.c_char_p, []),
    ("lbm_abi_version", C.c_int, []),
    ("lbm_device_count", C.c_int, [C.POINTER(C.c_int)]),
    ("lbm_create", C.c_int, [C.POINTER(LbmDesc), C.POINTER(P)]),
    ("lbm_copy_bandwidth", C.c_int, [I32, I32, I64, I32, I32, PD]),
    ("lbm_destroy", None, [P]),
    ("lbm_set_geometry", C.c_int, [P, P, P, P, P, P, P, P, P, I32]),
    ("lbm_init_equilibrium", C.c_int, [P, P, P, P, P, D, D, D, D]),
    ("lbm_step", C.c_int, [P, I64]),
    ("lbm_step_async", C.c_int, [P, I64]),
    ("lbm_synchronize", C.c_int, [P]),
    ("lbm_set_omega", C.c_int, [P, D]),
    ("lbm_get_macroscopic", C.c_int, [P, P, P, P, P]),
    ("lbm_get_macroscopic_box", C.c_int, [P, P, P, P, P, P, P]),
    ("lbm_check_finite", C.c_int, [P, C.POINTER(I32), P]),
    ("lbm_total_mass", C.c_int, [P, PD]),
    ("lbm_get_pdf", C.c_int, [P, I32, P]),
    ("lbm_set_pdf", C.c_int, [P, I32, P]),
    ("lbm_get_field", C.c_int, [P, I32, P]),
    ("lbm_set_field", C.c_int, [P, I32, P]),
    ("lbm_get_slot_of", C.c_int, [P, P]),
    ("lbm_get_flags", C.c_int, [P, P]),
    ("lbm_get_tile_index", C.c_int, [P, P, P, C.POINTER(I64)]),
    ("lbm_get_stats", C.c_int, [P, C.POINTER(LbmStats)]),
    ("lbm_halo_export", C.c_int, [P, P, C.POINTER(C.c_size_t)]),
    ("lbm_halo_connect", C.c_int, [P, P, P]),
    ("lbm19_feq", C.c_int, [I32, D, PD, PD]),
    ("lbm19_moments", C.c_int, [I32, PD, PD, PD]),
    ("lbm19_collide", C.c_int, [I32, PD, D, PD]),
    ("lbm19_zou_he_velocity", C.c_int, [I32, PD, I32, PD, PD]),
    ("lbm19_zou_he_pressure", C.c_int, [I32, PD, I32, D, PD]),
]


class LbmError(RuntimeError):
    def __init__(self, code, message):
        self.code = code
        super().__init__(message)


_lib = None


def load():
    """Load liblbm19.so; raise ImportError (loudly) when it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with "
            "`python -m paper_2108_13241_b200.build` (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.lbm_abi_version() != ABI_VERSION:
        raise ImportError("liblbm19.so ABI version mismatch; rebuild it")
    _lib = lib
    return lib


def last_error():
    return load().lbm_last_error().decode(errors="replace")


def check(rc, what=""):
    """Map a C return code onto the reference's exception types."""
    if rc == LBM_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == LBM_EINVAL:
        raise ValueError(msg)
    if rc == LBM_ESTATE:
        raise RuntimeError(msg)
    if rc == LBM_ENOMEM:
        raise MemoryError(msg)
    raise LbmError(rc, msg)


def ptr(a):
    """Raw data pointer of a C-contiguous numpy array (None passes NULL)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return a.ctypes.data_as(C.c_void_p)


def dptr(a):
    return a.ctypes.data_as(PD)


def device_count():
    n = C.c_int(0)
    rc = load().lbm_device_count(C.byref(n))
    if rc != 0:
        return 0
    return int(n.value)


def scalar_call(name, dtype, *args):
    """Helper for the lbm19_* scalar functions (host math, same source as the
    device kernel)."""
    return getattr(load(), name)(LBM_F32 if np.dtype(dtype) == np.float32 else LBM_F64, *args)
