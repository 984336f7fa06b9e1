"""CPU: the C-ABI library builds/loads and exports every symbol include/*.h declares."""
import ctypes
import glob
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = re.sub(r"/\*.*?\*/", "", open(h).read(), flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s+([A-Za-z_][A-Za-z0-9_]*)\s*\(",
                             src, flags=re.M):
            names.add(m.group(1))
    return names


def test_header_declares_the_boundary():
    names = _declared()
    for n in ["sl_setup", "fracop_apply", "precond_apply", "cp_dot", "cp_truncate", "pcg_solve"]:
        assert n in names


def test_library_exports_all_symbols():
    from paper_2006_09314_b200 import build
    from paper_2006_09314_b200.binding import ENTRY_POINTS
    path = build.build()
    lib = ctypes.CDLL(path)          # loading needs only libcudart, no device
    for name in sorted(_declared()):
        assert hasattr(lib, name), name
    assert set(ENTRY_POINTS) == _declared()
