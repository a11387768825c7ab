"""The C-ABI library loads on a CPU-only machine and exports exactly what
include/isaac_b200.h declares; ctypes struct layouts match the native ones.
No compute entry point is called here (no GPU)."""

import ctypes as C
import os
import re

import pytest

from paper_1611_09048_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "isaac_b200.h")


def declared_symbols():
    with open(HEADER) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"ISC_API\s+[\w\s\*]+?\b(isc_\w+)\s*\(", text)))


def test_header_declares_the_bound_symbols():
    decl = declared_symbols()
    assert len(decl) >= 19
    assert sorted(_abi.EXPORTED) == decl


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_abi.LIB_PATH):
        pytest.skip("library not built")
    lib = C.CDLL(_abi.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_struct_layouts_and_version():
    if not os.path.exists(_abi.LIB_PATH):
        pytest.skip("library not built")
    lib = _abi.lib()            # loads, checks version and every struct size
    assert lib.isc_abi_version() == _abi.ABI_VERSION
    assert lib.isc_flag_words() >= 10
    for which, st in enumerate((_abi.RenderArgs, _abi.Source, _abi.Camera, _abi.ClipPlane, _abi.ChainStep,
                                _abi.SwapArgs, _abi.ToyArgs)):
        assert lib.isc_struct_size(which) == C.sizeof(st)


def test_argument_validation_without_device():
    """Host-side validation in the library rejects bad blocks before any launch."""
    if not os.path.exists(_abi.LIB_PATH):
        pytest.skip("library not built")
    lib = _abi.lib()
    a = _abi.RenderArgs()
    assert lib.isc_render_local(C.byref(a), None) == 4          # SceneError: image size
    a.camera.width, a.camera.height = 4, 4
    assert lib.isc_render_local(C.byref(a), None) == 4          # step must be positive
    a.step = 0.5
    assert lib.isc_render_local(C.byref(a), None) == 1          # FieldError: sizes
    with pytest.raises(_abi.errors.FieldError):
        _abi.check(lib.isc_render_local(C.byref(a), None))
    a.brick_size[:] = [4, 4, 4]
    a.volume_size[:] = [4, 4, 4]
    a.decomposition[:] = [1, 1, 1]
    assert lib.isc_gradient_normals(C.byref(a), None, None, 1, None, None) == 7   # ValueError: no source in src[0]
    s = _abi.SwapArgs()
    s.size, s.rank, s.n_ctas, s.epoch = 3, 0, 1, 1
    assert lib.isc_binary_swap(C.byref(s), None) == 5           # CompositeError: not a power of two


def test_product_path_fails_loudly_without_library(monkeypatch, tmp_path):
    monkeypatch.setattr(_abi, "_lib", None)
    monkeypatch.setattr(_abi, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(_abi.NativeLibraryMissing):
        _abi.lib()


def test_integration_stub_matches_library():
    """The ctypes stub a reference maintainer would paste
    has the library's struct layouts and ABI version."""
    if not os.path.exists(_abi.LIB_PATH):
        pytest.skip("library not built")
    with open(os.path.join(ROOT, "INTEGRATION.md")) as fh:
        text = fh.read()
    code = text[text.index("class ChainStep"):text.index("# inside the reference's render_local")]
    ns = {"C": C, "lib": C.CDLL(_abi.LIB_PATH)}
    exec(code, ns)     # runs the stub's own asserts (version, struct sizes)
