"""CPU: the C-ABI library builds for sm_100a, loads, exports every symbol include/*.h declares,
and validates configurations exactly like LadderConfig::validate (config.hpp:74-96) before
touching the GPU. No compute calls (there is no GPU here)."""
import ctypes as C
import glob
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    from paper_1604_01946_b200 import _lib
    return _lib.load()


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(rw_[a-z0-9_]+)\s*\(", src))
    return sorted(names)


def test_library_exports_every_declared_symbol():
    L = _lib()
    syms = declared_symbols()
    assert len(syms) >= 15
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    from paper_1604_01946_b200 import _lib as mod
    assert sorted(mod.EXPORTS) == syms


def test_library_is_sm100a_tcgen05():
    """The shipped library carries sm_100a SASS with tcgen05 MMA, TMEM loads and TMA."""
    from paper_1604_01946_b200 import _lib as mod
    _lib()
    out = subprocess.run(["cuobjdump", "-sass", mod.lib_path()], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    sass = out.stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", mod.lib_path()], capture_output=True,
                                       text=True).stdout
    assert "UTCHMMA" in sass or "UTCMMA" in sass
    assert "UTMALDG" in sass
    assert "LDTM" in sass


def _cfg(**kw):
    from paper_1604_01946_b200 import _lib as mod
    base = dict(layers=2, hidden=8, input=8, batch=2, steps=4, cell_kind=3, opt_level=6,
                batch_steps=2, workers=2, seed=1, precision=0, schedule=0)
    base.update(kw)
    return mod.rw_config(**base)


@pytest.mark.parametrize("kw,msg", [
    (dict(opt_level=7), "opt_level must be in 0..6"),
    (dict(hidden=0), "hidden must be positive"),
    (dict(batch_steps=5), "batch_steps 5 exceeds steps 4"),
    (dict(cell_kind=7), "cell kind must be 0 (rnn-tanh), 1 (rnn-relu), 2 (gru) or 3 (lstm), got 7"),
    (dict(workers=0), "workers must be positive"),
])
def test_create_validates_like_reference(kw, msg):
    L = _lib()
    h = C.c_void_p()
    st = L.rw_create(C.byref(_cfg(**kw)), 0, C.byref(h))
    assert st == 1  # RW_EINVAL
    assert msg in L.rw_create_error().decode()
    assert not h.value


def test_flop_count_abi():
    assert _lib().rw_flop_count_cell(512, 512, 64) == 268435456


def test_python_config_validation_messages():
    from paper_1604_01946_b200 import Engine, LadderConfig
    with pytest.raises(ValueError, match="opt_level must be in 0..6, got 7"):
        Engine(LadderConfig(opt_level=7))
    with pytest.raises(ValueError, match="cell kind must be"):
        Engine(LadderConfig(kind=5))
