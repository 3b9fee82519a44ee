"""The C-ABI library loads and exports every symbol include/mlb.h declares
(no compute calls: this runs without a GPU)."""

import ctypes
import os
import re

import pytest

from paper_2409_16781_b200 import _cabi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mlb.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mlb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_what_the_binding_binds():
    assert declared_symbols() == sorted(_cabi.SYMBOLS)


def test_library_exports_every_declared_symbol():
    assert os.path.exists(_cabi.LIB_PATH), "run __graft_entry__.build() first"
    lib = ctypes.CDLL(_cabi.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_abi_version_and_layout_query():
    lib = _cabi.lib()
    assert lib.mlb_abi_version() == _cabi.ABI_VERSION
    lay = _cabi.Layout()
    _cabi.check(lib.mlb_layout_query(512, 512, 512, _cabi.MLB_F32, ctypes.byref(lay)))
    assert (lay.xp, lay.plane, lay.pop) == (512, 512 * 512, 514 * 512 * 512)
    assert lay.bytes == 19 * 514 * 512 * 512 * 4
    _cabi.check(lib.mlb_layout_query(9, 7, 5, _cabi.MLB_F64, ctypes.byref(lay)))
    assert lay.xp == 16 and lay.itemsize == 8  # 9 doubles -> one 128-byte line
    _cabi.check(lib.mlb_layout_query(33, 2, 1, _cabi.MLB_F32, ctypes.byref(lay)))
    assert lay.xp == 64


def test_errors_map_to_reference_exception_types():
    lib = _cabi.lib()
    lay = _cabi.Layout()
    with pytest.raises(ValueError, match="dtype"):
        _cabi.check(lib.mlb_layout_query(8, 8, 8, 7, ctypes.byref(lay)))
    with pytest.raises(ValueError, match="empty"):
        _cabi.check(lib.mlb_layout_query(0, 8, 8, 0, ctypes.byref(lay)))
    with pytest.raises(ValueError, match="NULL"):
        _cabi.check(lib.mlb_step(None, None, None, None))


def test_device_layout_mirror_matches_the_library():
    from paper_2409_16781_b200.fields import DeviceLayout
    lib = _cabi.lib()
    lay = _cabi.Layout()
    for (nx, ny, nz, code, sz) in [(512, 512, 512, 0, 4), (9, 7, 5, 1, 8), (100, 3, 2, 0, 4),
                                   (1024, 512, 64, 1, 8)]:
        _cabi.check(lib.mlb_layout_query(nx, ny, nz, code, ctypes.byref(lay)))
        m = DeviceLayout(nx, ny, nz, sz)
        assert (m.xp, m.plane, m.pop, m.total) == (lay.xp, lay.plane, lay.pop, lay.total)


def test_no_contracted_multiply_adds_in_the_device_code():
    """Bit-exact parity rests on every floating-point operation being one IEEE
    rounding.  -fmad=false keeps nvcc / ptxas from contracting scalar a*b+c,
    but ptxas 12.9 contracts PACKED fp32 multiplies and adds (mul.rn.f32x2 +
    add.rn.f32x2 -> FFMA2) regardless - which once cost a half-ulp in one of
    ~20 000 values of the fp16-storage kernels.  Guard: in the built library
    the only packed FMAs are the exact a - b = FFMA2(b, -1, a) form, and the
    only scalar FMAs are those of the IEEE division / reciprocal sequences."""
    import shutil
    import subprocess
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump) or not os.path.exists(_cabi.LIB_PATH):
        pytest.skip("cuobjdump or the built library is not available")
    sass = subprocess.run([cuobjdump, "-sass", _cabi.LIB_PATH], capture_output=True,
                          text=True, check=True).stdout
    packed = [ln for ln in sass.splitlines() if " FFMA2 " in ln]
    assert packed, "expected the packed-fp32 collide in the fp16-storage kernels"
    bad = [ln.strip() for ln in packed if ", -1, " not in ln]
    assert not bad, bad[:5]
    # scalar kernels: count FFMA per kernel; the fused step kernels in fp32 may
    # only contain the handful that belong to the division sequence (1 / rho)
    per_kernel, name = {}, None
    for ln in sass.splitlines():
        if "Function :" in ln:
            name = ln.split("Function :")[1].strip()
            per_kernel[name] = 0
        elif name and (" FFMA " in ln or " DFMA " in ln):
            per_kernel[name] += 1
    for name, n in per_kernel.items():
        if "step_" in name or "aa_" in name:
            # one division per cell of a pack: <= 8 packs' worth of Newton steps
            assert n <= 80, (name, n)
