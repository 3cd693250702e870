"""ctypes binding of librfb.so (the C ABI declared in include/rfb.h).

There is no CPU fallback: if the extension is missing or cannot be loaded,
every entry point raises ``ExtensionMissing``; a non-zero return code raises
``DeviceError`` with the library's message.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import DeviceError, ExtensionMissing

ABI_VERSION = 15  # include/rfb.h RFB_ABI_VERSION
_lock = threading.Lock()
_lib = None

c_double_p = ctypes.POINTER(ctypes.c_double)


class rfb_scene(ctypes.Structure):
    _fields_ = [
        ("n_sites", ctypes.c_int64),
        ("n_edges", ctypes.c_int64),
        ("site4", ctypes.c_void_p),
        ("offsets", ctypes.c_void_p),
        ("neighbors", ctypes.c_void_p),
        ("sh", ctypes.c_void_p),
        ("cells", ctypes.c_void_p),
        ("edges", ctypes.c_void_p),
        ("edge_nbr", ctypes.c_void_p),
        ("sh32", ctypes.c_void_p),
        ("packed", ctypes.c_int32),
        ("sh_absmax", ctypes.c_float),
        ("sh_degree", ctypes.c_int32),
        ("positions_f64", ctypes.c_int32),
        ("background", ctypes.c_double * 3),
        ("sh_absmax_dev", ctypes.c_void_p),
        ("pk_of", ctypes.c_void_p),
        ("pk_id", ctypes.c_void_p),
        ("view_rx", ctypes.c_int32),
        ("view_ry", ctypes.c_int32),
    ]


class rfb_params(ctypes.Structure):
    _fields_ = [
        ("epsilon", ctypes.c_double),
        ("width_floor", ctypes.c_double),
        ("step_limit", ctypes.c_int32),
        ("lanes_per_ray", ctypes.c_int32),
    ]


class rfb_rays(ctypes.Structure):
    _fields_ = [
        ("m", ctypes.c_int64),
        ("origins", ctypes.c_void_p),
        ("directions", ctypes.c_void_p),
        ("t_min", ctypes.c_void_p),
        ("t_max", ctypes.c_void_p),
        ("start_sites", ctypes.c_void_p),
        ("order", ctypes.c_void_p),
        ("region", ctypes.c_void_p),
    ]


class rfb_fwd_out(ctypes.Structure):
    _fields_ = [
        ("rgb", ctypes.c_void_p),
        ("residual", ctypes.c_void_p),
        ("wsum", ctypes.c_void_p),
        ("status", ctypes.c_void_p),
        ("nseg", ctypes.c_void_p),
        ("ray_counters", ctypes.c_void_p),
        ("counters", ctypes.c_void_p),
        ("f64_outputs", ctypes.c_int32),
        ("seg_capacity", ctypes.c_int32),
        ("seg_cells", ctypes.c_void_p),
        ("seg_t0", ctypes.c_void_p),
        ("seg_t1", ctypes.c_void_p),
        ("seg_first", ctypes.c_int64),
        ("seg_count", ctypes.c_int64),
    ]


class rfb_grads(ctypes.Structure):
    _fields_ = [("site4g", ctypes.c_void_p), ("sh", ctypes.c_void_p)]


class rfb_locate_grid(ctypes.Structure):
    _fields_ = [
        ("lo", ctypes.c_double * 3),
        ("cell", ctypes.c_double),
        ("dims", ctypes.c_int32 * 3),
        ("pad_", ctypes.c_int32),
        ("hint", ctypes.c_void_p),
    ]


class rfb_camera(ctypes.Structure):
    _fields_ = [
        ("pose", ctypes.c_double * 16),
        ("width", ctypes.c_int32),
        ("height", ctypes.c_int32),
        ("focal", ctypes.c_double),
        ("cx", ctypes.c_double),
        ("cy", ctypes.c_double),
        ("kind", ctypes.c_int32),
        ("pad_", ctypes.c_int32),
    ]


P = ctypes.POINTER
VP = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32
F64 = ctypes.c_double
SZ = ctypes.c_size_t

# name -> (restype, argtypes); must match include/rfb.h exactly.
SIGNATURES = {
    "rfb_abi_version": (ctypes.c_int, []),
    "rfb_error_string": (ctypes.c_char_p, [ctypes.c_int]),
    "rfb_device_ok": (ctypes.c_int, []),
    "rfb_host_device_pointer": (ctypes.c_int, [VP, P(VP)]),
    "rfb_pack_scene": (ctypes.c_int, [VP, VP, VP, VP, VP, I64, I64, VP, VP, VP, VP, VP, VP, VP,
                                      VP, VP, I32, VP]),
    "rfb_softplus": (ctypes.c_int, [VP, I64, VP, VP, VP, VP, VP]),
    "rfb_camera_rays": (ctypes.c_int, [P(rfb_camera), I64, I64, VP, VP]),
    "rfb_post_grad_adam": (ctypes.c_int, [I64, VP, VP, VP, VP, VP, F64, I32, I32, VP, VP, VP, VP, VP]),
    "rfb_refresh_scene": (ctypes.c_int, [P(rfb_scene), VP, VP, I32, VP]),
    "rfb_locate": (ctypes.c_int, [P(rfb_scene), VP, I64, I32, VP, VP]),
    "rfb_build_locate_grid": (ctypes.c_int, [P(rfb_scene), P(rfb_locate_grid), VP]),
    "rfb_locate_seeded": (ctypes.c_int, [P(rfb_scene), VP, I64, P(rfb_locate_grid), I32, VP, VP]),
    "rfb_adjacency_workspace_bytes": (SZ, [I64, I32]),
    "rfb_build_adjacency": (ctypes.c_int, [VP, I64, I32, VP, VP, I64, VP, P(ctypes.c_int64), VP,
                                           SZ, VP]),
    "rfb_adjacency_emit": (ctypes.c_int, [I64, I32, VP, VP, VP, VP, SZ, VP]),
    "rfb_sh_basis": (ctypes.c_int, [VP, I64, VP, VP]),
    "rfb_cell_colors": (ctypes.c_int, [VP, VP, VP, I64, VP, VP, VP]),
    "rfb_composite_segments": (ctypes.c_int, [VP, VP, VP, I64, VP, VP, VP, VP,
                                              P(ctypes.c_double), VP, VP, VP, VP]),
    "rfb_segments_workspace_bytes": (SZ, [I64, I64]),
    "rfb_face_t_gradients": (ctypes.c_int, [VP, VP, VP, VP, VP, VP, I64, VP, VP]),
    "rfb_backward_segments": (ctypes.c_int, [VP, VP, VP, P(ctypes.c_double), VP, VP, VP, VP,
                                             I64, VP, VP, VP, VP, VP, VP, VP, VP, SZ, VP]),
    "rfb_quantile_segments": (ctypes.c_int, [VP, VP, VP, VP, I64, VP, VP, VP, VP, VP, I32,
                                             ctypes.c_double, ctypes.c_double, VP, VP, VP, VP,
                                             SZ, VP]),
    "rfb_effect_rays": (ctypes.c_int, [VP, VP, VP, I64, P(ctypes.c_double), I32, ctypes.c_double,
                                       VP, VP, VP]),
    "rfb_render_rays": (ctypes.c_int, [P(rfb_scene), P(rfb_rays), P(rfb_params), P(rfb_fwd_out),
                                       VP, SZ, VP]),
    "rfb_render_image": (ctypes.c_int, [P(rfb_scene), P(rfb_camera), P(rfb_params), F64, F64, I32,
                                        VP, I64, I32, I32, P(rfb_fwd_out), VP, SZ, VP]),
    "rfb_workspace_bytes": (SZ, [I64, I32, I32]),
    "rfb_cull_scene": (ctypes.c_int, [P(rfb_scene), P(ctypes.c_double), I32, VP, VP, P(rfb_scene),
                                      VP]),
    "rfb_cull_view": (ctypes.c_int, [P(rfb_scene), P(rfb_camera), I32, I32, VP, VP, P(rfb_scene),
                                     VP]),
    "rfb_backward_rays": (ctypes.c_int, [P(rfb_scene), P(rfb_rays), P(rfb_params), VP,
                                         P(rfb_fwd_out), P(rfb_grads), VP, SZ, VP]),
    "rfb_train_batch": (ctypes.c_int, [P(rfb_scene), P(rfb_rays), P(rfb_params), VP, F64, F64, VP,
                                       I32, F64, P(rfb_fwd_out), P(rfb_grads), VP, VP, SZ, VP]),
}


def lib_path() -> str:
    return os.environ.get("RFB_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                  "librfb.so"))


def load(path: str | None = None):
    """Load (once) and type the C ABI.  Raises ExtensionMissing."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = path or lib_path()
        if not os.path.exists(p):
            raise ExtensionMissing(
                f"{p} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        try:
            lib = ctypes.CDLL(p)
        except OSError as e:  # pragma: no cover - depends on the box
            raise ExtensionMissing(f"cannot load {p}: {e}") from e
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.rfb_abi_version() != ABI_VERSION:
            raise ExtensionMissing("librfb.so ABI version mismatch; rebuild")
        if path is None:
            _lib = lib
        return lib


def check(code: int, what: str):
    if code != 0:
        msg = load().rfb_error_string(code).decode()
        raise DeviceError(f"{what} failed: {msg} (code {code})")
