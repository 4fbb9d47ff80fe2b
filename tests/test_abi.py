"""The C-ABI library loads and exports every symbol include/*.h declares (CPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:spd_status|void|const char\*|int|long long)\s+(\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_headers_declare_the_north_star_entry_points():
    names = _declared("spdhss.h")
    for n in ["h2_build", "spdhss_build", "hss_solve", "h2_matvec", "pcg_solve", "spd_query",
              "spd_comm_init", "h2_free", "hss_free", "spd_last_error"]:
        assert n in names


def test_library_exports_every_declared_symbol():
    import paper_2011_07632_b200 as spd
    if not os.path.exists(spd.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    lib = ctypes.CDLL(spd.LIB_PATH)
    for h in ("spdhss.h", "spdhss_testing.h"):
        for n in _declared(h):
            assert hasattr(lib, n), f"{n} declared in {h} but not exported"
    spd.lib()   # binding signatures resolve


def test_binding_fails_loudly_without_library(tmp_path, monkeypatch):
    import paper_2011_07632_b200 as spd
    monkeypatch.setattr(spd, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(spd, "_lib", None)
    with pytest.raises(ImportError):
        spd.lib()
