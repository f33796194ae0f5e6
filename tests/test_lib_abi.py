"""CPU checks of the C-ABI library: it loads, exports every symbol include/topt.h declares,
validates parameters without touching a GPU, and the ctypes structs match the header."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "topt.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(topt_[a-z_0-9]+)\s*\(", src)))


def test_header_symbols_exported_and_bound():
    from paper_2510_08782_b200 import _lib
    names = _declared()
    assert "topt_eval_gradient" in names and "topt_solve" in names
    for n in names:
        assert hasattr(_lib.LIB, n), n
        assert n in _lib.SIGNATURES, n
    assert _lib.LIB.topt_abi_version() == 1


def test_param_validation_without_gpu():
    from paper_2510_08782_b200 import Config, _lib
    LIB = _lib.LIB
    ctx = ctypes.c_void_p()
    bad = [
        Config(n=(64, 63), nt=4),                 # odd
        Config(n=(64, 64), nt=4, alpha=0.0),      # alpha <= 0
        Config(n=(64, 64), nt=4, sigma=0),        # sigma < 1
        Config(n=(64, 64), nt=0),                 # nt < 1
        Config(n=(64, 64, 64), nt=4, tau=-1),
    ]
    for cfg in bad:
        p = cfg.params()
        assert LIB.topt_create(ctypes.byref(p), 0, 1, None, 0, ctypes.byref(ctx)) == -1
    p = Config(n=(96, 64), nt=4).params()   # even but not a power of two
    assert LIB.topt_create(ctypes.byref(p), 0, 1, None, 0, ctypes.byref(ctx)) == -2
    # z-slab decomposition parameter checks (world > 1)
    p = Config(n=(64, 64, 64), nt=4).params()
    assert LIB.topt_create(ctypes.byref(p), 0, 3, None, 0, ctypes.byref(ctx)) == -1      # world not 2^k
    p = Config(n=(64, 64, 16), nt=4).params()
    assert LIB.topt_create(ctypes.byref(p), 0, 8, None, 0, ctypes.byref(ctx)) == -1      # nz/P < halo 4
    p = Config(n=(64, 64), nt=4).params()
    assert LIB.topt_create(ctypes.byref(p), 0, 2, None, 0, ctypes.byref(ctx)) == -1      # 2D on 2 ranks
    p = Config(n=(16, 64, 64), nt=4).params()
    assert LIB.topt_create(ctypes.byref(p), 0, 2, None, 0, ctypes.byref(ctx)) == -2      # nx < 32 tiles
    p = Config(n=(64, 64, 64), nt=4).params()
    assert LIB.topt_create(ctypes.byref(p), 1, 2, None, 0, ctypes.byref(ctx)) == -1      # emulation runs as rank 0
    assert b"" != LIB.topt_last_error()


def test_struct_layout_matches_header(tmp_path):
    """ctypes Params/Report offsets equal the C compiler's offsetof for include/topt.h."""
    import subprocess
    from paper_2510_08782_b200 import _lib
    checks = []
    for cname, cls in (("topt_params", _lib.Params), ("topt_report", _lib.Report)):
        checks.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in cls._fields_:
            checks.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    src = tmp_path / "layout.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "topt.h"\nint main(void){' + "".join(checks)
                   + "return 0;}\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l}
    for cname, cls in (("topt_params", _lib.Params), ("topt_report", _lib.Report)):
        assert got[(cname, "size")] == ctypes.sizeof(cls)
        for f, _ in cls._fields_:
            assert got[(cname, f)] == getattr(cls, f).offset, (cname, f)
