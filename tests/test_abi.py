"""The C-ABI library (no GPU needed): it loads, exports every symbol declared
in include/rfb.h, its struct layouts match the ctypes mirror, and argument
validation fails loudly (RFB_EINVAL) before any device work."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2502_01157_b200 import _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "rfb.h")


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char \*)\s*(rfb_\w+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2502_01157_b200 import _build

    _build.build_extension()
    return _lib.load()


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.SIGNATURES), "ctypes signature table out of sync with rfb.h"
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.lib_path()], capture_output=True,
                         text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", out), f"{n} not exported"


def test_abi_version_and_errors(lib):
    assert lib.rfb_abi_version() == 15
    assert lib.rfb_error_string(0) == b"ok"
    assert lib.rfb_error_string(-1) == b"invalid argument"


def _c_layout():
    """sizeof/offsetof of the ABI structs as the C compiler sees them."""
    prog = r'''
#include <stdio.h>
#include <stddef.h>
#include "rfb.h"
#define F(T, m) printf(#T "." #m " %zu\n", offsetof(T, m));
int main(void) {
  printf("rfb_scene %zu\nrfb_params %zu\nrfb_rays %zu\nrfb_fwd_out %zu\nrfb_grads %zu\nrfb_camera %zu\n",
         sizeof(rfb_scene), sizeof(rfb_params), sizeof(rfb_rays), sizeof(rfb_fwd_out),
         sizeof(rfb_grads), sizeof(rfb_camera));
  F(rfb_scene, sh32) F(rfb_scene, packed) F(rfb_scene, sh_absmax) F(rfb_scene, background)
  F(rfb_scene, sh_absmax_dev) F(rfb_scene, view_ry) F(rfb_rays, region)
  F(rfb_fwd_out, f64_outputs) F(rfb_fwd_out, seg_t1) F(rfb_fwd_out, seg_count) F(rfb_camera, focal) F(rfb_params, lanes_per_ray)
  return 0;
}
'''
    import tempfile

    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "l.c")
        open(c, "w").write(prog)
        exe = os.path.join(d, "l")
        subprocess.run(["gcc", "-I", os.path.dirname(HEADER), c, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    return dict(line.rsplit(" ", 1) for line in out.strip().splitlines())


def test_struct_layout_matches_ctypes():
    lay = {k: int(v) for k, v in _c_layout().items()}
    for name in ["rfb_scene", "rfb_params", "rfb_rays", "rfb_fwd_out", "rfb_grads", "rfb_camera"]:
        assert ctypes.sizeof(getattr(_lib, name)) == lay[name], name
    for key, val in lay.items():
        if "." in key:
            s, m = key.split(".")
            assert getattr(getattr(_lib, s), m).offset == val, key


def test_argument_validation_without_device(lib):
    p = _lib.rfb_params()
    p.step_limit = 4096
    rays = _lib.rfb_rays()
    out = _lib.rfb_fwd_out()
    assert lib.rfb_render_rays(None, ctypes.byref(rays), ctypes.byref(p), ctypes.byref(out), None,
                               0, None) == -1
    sc = _lib.rfb_scene()  # all-NULL scene is rejected
    assert lib.rfb_render_rays(ctypes.byref(sc), ctypes.byref(rays), ctypes.byref(p),
                               ctypes.byref(out), None, 0, None) == -1
    cam = _lib.rfb_camera()
    assert lib.rfb_camera_rays(ctypes.byref(cam), 0, 1, None, None) == -1
    assert lib.rfb_pack_scene(None, None, None, None, None, 0, 0, None, None, None, None, None,
                              None, None, None, None, 0, None) == -1
    assert lib.rfb_softplus(None, 1, None, None, None, None, None) == -1
    assert lib.rfb_host_device_pointer(None, None) == -1
    view = _lib.rfb_scene()
    dirs = (ctypes.c_double * 3)(0.0, 0.0, -1.0)
    assert lib.rfb_cull_scene(ctypes.byref(sc), dirs, 1, None, None, ctypes.byref(view), None) == -1
    assert lib.rfb_cull_scene(None, dirs, 1, None, None, ctypes.byref(view), None) == -1
