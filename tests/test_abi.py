"""The C ABI library builds for sm_100a, loads, and exports every entry point that
include/mk.h declares.  No GPU needed (no compute calls)."""
import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def libmk():
    # by path: importing the package would load the library before it is built
    import importlib.util
    spec = importlib.util.spec_from_file_location("_mk_build", ROOT / "paper_1904_08755_b200" / "build.py")
    build = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(build)
    return build.build()


def _declared():
    hdr = (ROOT / "include" / "mk.h").read_text()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(mk_[a-z_0-9]+)\s*\(", hdr)))


def test_header_declares_entry_points():
    names = _declared()
    for must in ("mk_coords_quantize", "mk_coords_create", "mk_coords_stride", "mk_kmap_build",
                 "mk_conv_forward", "mk_conv_backward", "mk_conv_transpose_forward", "mk_conv_transpose_backward"):
        assert must in names


def test_library_exports_every_declared_symbol(libmk):
    lib = ctypes.CDLL(str(libmk))
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a(libmk):
    out = subprocess.run(["cuobjdump", "--list-elf", str(libmk)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_binding_mirrors_abi_names(libmk):
    from paper_1904_08755_b200 import _lib
    assert set(_lib.EXPORTS) == set(_declared())


def test_region_offsets_without_gpu(libmk):
    # mk_region_offsets is host-only: check it against the paper's counts.
    import numpy as np
    import paper_1904_08755_b200 as mk
    assert mk.region_offsets(mk.Region(mk.HYPERCUBE, 4, 5)).shape == (625, 4)
    assert mk.region_offsets(mk.Region(mk.HYBRID, 4, 3)).shape == (29, 4)
    assert mk.region_offsets(mk.Region(mk.HYPERCROSS, 3, 3)).shape == (7, 3)
    assert mk.region_offsets(mk.Region(mk.HYPERCUBE, 1, 3)).ravel().tolist() == [-1, 0, 1]
    custom = np.array([[1, 0], [0, 0]], np.int32)
    assert mk.region_offsets(mk.Region(mk.CUSTOM, 2, offsets=custom)).tolist() == custom.tolist()
    with pytest.raises(mk.MkError):
        mk.region_offsets(mk.Region(mk.CUSTOM, 2, offsets=np.array([[0, 0], [0, 0]])))


@pytest.mark.parametrize("kind,D,size,dil", [(0, 3, 3, 1), (0, 3, 2, 1), (0, 4, 5, 1), (1, 3, 3, 1), (1, 4, 3, 2),
                                             (2, 4, 3, 1), (2, 4, 5, 1), (0, 2, [3, 5], [2, 1]), (0, 1, 7, 3)])
def test_region_offsets_match_oracle(libmk, orc, kind, D, size, dil):
    # Both are host code; the library's enumeration must equal the oracle's (R2-R4).
    import paper_1904_08755_b200 as mk
    got = mk.region_offsets(mk.Region(kind, D, size, dil))
    want = orc.region(kind, D, size if isinstance(size, list) else [size] * D,
                      dil if isinstance(dil, list) else [dil] * D)
    assert got.tolist() == want.tolist()
