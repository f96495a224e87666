"""CPU: the reference's binary parameter file (param_io.hpp) -- a fixture written by the
unmodified reference (tests/golden/make_param_file.cpp) loads bit-exactly and equals our
init_params restatement; save/load round trips; the reference's error messages."""
import os
import struct
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_01946_b200 import LadderConfig, init_params  # noqa: E402
from paper_1604_01946_b200 import param_io  # noqa: E402

FIX = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "params_lstm_L2H5I7.bin")


def _cfg():
    return LadderConfig(layers=2, hidden=5, input=7, batch=3, steps=4, seed=11)


def test_reference_written_file_loads_bit_exact():
    h, params = param_io.load_params(FIX)
    assert (h.kind, h.layers, h.hidden, h.input, h.batch_hint) == (3, 2, 5, 7, 3)
    assert os.path.getsize(FIX) == param_io.param_file_size(h)
    ours = init_params(_cfg())
    for a, b in zip(params, ours):
        assert np.array_equal(a.w, b.w) and np.array_equal(a.r, b.r)
        assert np.array_equal(a.bias, 0.01 * np.arange(1, 21, dtype=np.float32))
    param_io.check_matches(h, _cfg())


def test_save_load_round_trip_is_bitwise(tmp_path):
    h, params = param_io.load_params(FIX)
    out = tmp_path / "p.bin"
    param_io.save_params(str(out), h, params)
    assert out.read_bytes() == open(FIX, "rb").read()


def test_reference_error_messages(tmp_path):
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOTAFILE" + b"\0" * 40)
    with pytest.raises(RuntimeError, match="bad magic"):
        param_io.load_params(str(bad))
    data = open(FIX, "rb").read()
    trunc = tmp_path / "trunc.bin"
    trunc.write_bytes(data[:100])
    with pytest.raises(RuntimeError, match="truncated while reading layer 0 W"):
        param_io.load_params(str(trunc))
    kind = tmp_path / "kind.bin"
    kind.write_bytes(data[:16] + struct.pack("<I", 9) + data[20:])
    with pytest.raises(RuntimeError, match="unknown cell kind 9"):
        param_io.load_params(str(kind))
    h, _ = param_io.load_params(FIX)
    c = _cfg()
    c.hidden = 6
    with pytest.raises(RuntimeError, match="hidden size is 5 but the configuration expects 6"):
        param_io.check_matches(h, c)
    with pytest.raises(ValueError, match="header says 2 layers, got 1"):
        param_io.save_params(str(tmp_path / "x.bin"), h, init_params(_cfg())[:1])


@pytest.mark.gpu
def test_param_file_into_device_context_matches_reference(reference):
    """The loaded file drives a device context; results match the reference engine on the same
    parameters (fp32-parity tolerance)."""
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from parity import assert_within, compare, make_case, run_device, run_reference
    from oracle import Dims
    from paper_1604_01946_b200 import Engine
    h, params = param_io.load_params(FIX)
    c, _, x, dy, h0, c0 = make_case(Dims(h.layers, h.hidden, h.input, 3, 4), seed=11, bias=True, state=True)
    param_io.check_matches(h, c)
    eng = Engine(c, precision="fp32")
    params = eng.load_params_file(FIX)
    dev = run_device(eng, params, x, dy, h0, c0)
    ref = run_reference(reference, c, params, x, dy, h0, c0)
    assert_within(compare(dev, ref, c), "fp32")


def test_cpp_facade_param_io(tmp_path):
    """The C++ facade's rnnwave/param_io.hpp (include/) reads the reference-written file
    bit-exactly and writes it back byte-identically (tests/cpp/param_io_check.cpp)."""
    import shutil
    import subprocess
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "pio"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I" + os.path.join(root, "include"),
                    os.path.join(root, "tests", "cpp", "param_io_check.cpp"), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe), FIX, str(tmp_path / "out.bin")], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
