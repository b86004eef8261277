"""CPU-only checks of the C-ABI boundary: librade.so loads, exports every function that
include/rade.h declares, the ctypes mirrors match the header's structs, and argument
validation rejects bad calls before any CUDA work (no GPU needed for those paths)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rade.h")


@pytest.fixture(scope="module")
def native():
    from paper_2406_01467_b200 import build
    build.build()
    from paper_2406_01467_b200 import _native
    _native.load()
    return _native


def _declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(rd_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_four_stages():
    names = _declared_functions()
    for f in ("rd_preprocess", "rd_bin", "rd_render_fwd", "rd_render_bwd"):
        assert f in names


def test_library_exports_every_declared_symbol(native):
    names = _declared_functions()
    out = subprocess.run(["nm", "-D", "--defined-only", native.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(rd_\w+)\b", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    # and the Python binding binds exactly those names
    assert sorted(native.SIGNATURES) == names


def test_struct_layouts_match_header(native):
    """Sizes/offsets of the ctypes mirrors equal the C structs (compiled probe)."""
    probe = r"""
#include "rade.h"
#include <stddef.h>
#include <stdio.h>
int main(void) {
  printf("%zu %zu %zu %zu %zu\n", sizeof(rd_camera), sizeof(rd_options), sizeof(rd_gaussians), sizeof(rd_grads),
         sizeof(rd_stats));
  printf("%zu %zu %zu %zu %zu %zu\n", offsetof(rd_camera, znear), offsetof(rd_options, sh_degree),
         offsetof(rd_gaussians, sh), offsetof(rd_stats, key_bits), offsetof(rd_options, guard_band),
         offsetof(rd_stats, n_big));
  return 0;
}
"""
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "p.c")
        open(c, "w").write(probe)
        exe = os.path.join(d, "p")
        subprocess.check_call(["gcc", "-std=c99", f"-I{os.path.join(ROOT, 'include')}", c, "-o", exe])
        lines = subprocess.check_output([exe], text=True).split("\n")
    sizes = [int(x) for x in lines[0].split()]
    offs = [int(x) for x in lines[1].split()]
    assert sizes == [ctypes.sizeof(native.RdCamera), ctypes.sizeof(native.RdOptions),
                     ctypes.sizeof(native.RdGaussians), ctypes.sizeof(native.RdGrads), ctypes.sizeof(native.RdStats)]
    assert offs == [native.RdCamera.znear.offset, native.RdOptions.sh_degree.offset, native.RdGaussians.sh.offset,
                    native.RdStats.key_bits.offset, native.RdOptions.guard_band.offset, native.RdStats.n_big.offset]


def test_options_default_and_version(native):
    lib = native.load()
    o = native.RdOptions()
    assert lib.rd_options_default(ctypes.byref(o)) == 0
    assert o.tile == 16 and abs(o.alpha_min - 1 / 255) < 1e-9 and abs(o.alpha_max - 0.99) < 1e-7
    assert abs(o.T_min - 1e-4) < 1e-10 and o.median_T == 0.5 and abs(o.dilation - 0.3) < 1e-7 and o.sh_degree == 3
    assert o.guard_band == 0.0  # reading S6b off by default
    assert b"sm_100a" in lib.rd_version()
    assert lib.rd_options_default(None) == native.RD_ERR_INVALID_ARGUMENT


def _view(native):
    lib = native.load()
    keep = []

    def alloc(nbytes, ctx):
        raise AssertionError("no allocation expected on argument errors")

    a, f = native.ALLOC_FN(alloc), native.FREE_FN(lambda p, c: None)
    keep += [a, f]
    h = ctypes.c_void_p()
    assert lib.rd_view_create(ctypes.byref(h), a, f, None) == 0
    return lib, h, keep


def test_argument_validation_without_gpu(native):
    lib, h, keep = _view(native)
    cam = native.RdCamera(fx=10, fy=10, cx=5, cy=5, width=10, height=10, znear=0.2)
    opt = native.RdOptions()
    lib.rd_options_default(ctypes.byref(opt))
    g = native.RdGaussians(n=-1, sh_coeffs=16)
    assert lib.rd_preprocess(h, ctypes.byref(g), ctypes.byref(cam), ctypes.byref(opt), None) == 1
    assert b"n < 0" in lib.rd_last_error()
    g = native.RdGaussians(n=5, sh_coeffs=16)  # NULL arrays
    assert lib.rd_preprocess(h, ctypes.byref(g), ctypes.byref(cam), ctypes.byref(opt), None) == 1
    fake = ctypes.c_void_p(16)
    g = native.RdGaussians(5, 16, fake, fake, fake, fake, fake)
    for field, val in (("tile", 64), ("tile", 12), ("alpha_min", 0.0), ("alpha_max", 1.5), ("sh_degree", 4), ("T_min", -1.0),
                       ("guard_band", -0.1), ("guard_band", float("inf"))):
        o2 = native.RdOptions()
        lib.rd_options_default(ctypes.byref(o2))
        setattr(o2, field, val)
        assert lib.rd_preprocess(h, ctypes.byref(g), ctypes.byref(cam), ctypes.byref(o2), None) == 1, field
    o2 = native.RdOptions()
    lib.rd_options_default(ctypes.byref(o2))
    g4 = native.RdGaussians(5, 4, fake, fake, fake, fake, fake)  # degree-1 storage, degree-3 requested
    assert lib.rd_preprocess(h, ctypes.byref(g4), ctypes.byref(cam), ctypes.byref(o2), None) == 1
    cam0 = native.RdCamera(fx=10, fy=10, cx=5, cy=5, width=0, height=10, znear=0.2)
    assert lib.rd_preprocess(h, ctypes.byref(g), ctypes.byref(cam0), ctypes.byref(opt), None) == 1
    # the binning's per-axis tile histograms cap an image at 2047 tiles per axis (rade.h rd_bin)
    o8 = native.RdOptions()
    lib.rd_options_default(ctypes.byref(o8))
    o8.tile = 8
    big = native.RdCamera(fx=10, fy=10, cx=5, cy=5, width=8 * 2048, height=10, znear=0.2)
    assert lib.rd_preprocess(h, ctypes.byref(g), ctypes.byref(big), ctypes.byref(o8), None) == 1
    assert b"too large" in lib.rd_last_error()
    # out-of-order calls are state errors
    assert lib.rd_bin(h, None, None) == native.RD_ERR_STATE
    assert lib.rd_render_fwd(h, None, None, None, None, None) == native.RD_ERR_STATE
    gr = native.RdGrads()
    assert lib.rd_render_bwd(h, ctypes.byref(g), None, None, None, None, ctypes.byref(gr), None) == native.RD_ERR_STATE
    assert lib.rd_view_destroy(h) == 0
    assert lib.rd_view_create(None, native.ALLOC_FN(), native.FREE_FN(), None) == 1
    h2 = ctypes.c_void_p()
    a = native.ALLOC_FN(lambda n, c: None)
    assert lib.rd_view_create(ctypes.byref(h2), a, native.FREE_FN(), None) == 1  # alloc without free


def test_binding_refuses_missing_library(tmp_path):
    from paper_2406_01467_b200 import _native
    saved = _native._lib
    _native._lib = None
    try:
        with pytest.raises(ImportError):
            _native.load(str(tmp_path / "nope.so"))
    finally:
        _native._lib = saved


def test_product_path_does_not_import_oracle():
    """The product package never references oracle/ (test infrastructure only)."""
    pkg = os.path.join(ROOT, "paper_2406_01467_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src and "rade_oracle" not in src, f
