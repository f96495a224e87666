"""Generate tests/golden/lstm_golden.npz from the UNMODIFIED reference engine.

Run here (where /root/reference exists): python tests/golden/make_golden.py
The reference is compiled by oracle/Makefile into oracle/_ref/ (a shim that calls
rnnwave::Engine / init_params / verify::make_input); the fixtures pin the C restatement
(oracle/lstm_oracle.c) and, with tolerances, the GPU engine. Small shapes only (KBs).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

# (layers, hidden, input, batch, steps, seed, nonzero bias, initial state)
CASES = [
    (1, 1, 1, 1, 1, 11, False, False),
    (1, 5, 7, 3, 4, 42, False, False),
    (2, 8, 6, 2, 4, 17, True, False),   # test_engine.cpp:115-145 shape
    (2, 4, 4, 2, 3, 23, True, True),    # test_engine.cpp:164-190 shape (h0/c0)
    (3, 16, 12, 4, 6, 5, True, True),
    (2, 33, 20, 5, 3, 99, True, True),
]


def main():
    R = oracle.Reference()
    out = {}
    for ci, (L, H, I, B, T, seed, bias, state) in enumerate(CASES):
        d = oracle.Dims(L, H, I, B, T)
        w, r = R.init_params(d, seed)
        rs = oracle.Restatement()
        b = [rs.fill_symmetric(seed, 300 + l, 0.5, 4 * H) if bias else np.zeros(4 * H, np.float32)
             for l in range(L)]
        h0 = c0 = None
        if state:
            h0 = [rs.fill_symmetric(seed, 50 + l, 1.0, H * B).reshape((H, B), order="F") for l in range(L)]
            c0 = [rs.fill_symmetric(seed, 60 + l, 1.0, H * B).reshape((H, B), order="F") for l in range(L)]
        x = R.make_input(d, seed)
        dy = R.make_dy(d, seed)
        res = R.run(d, w, r, b, x, h0, c0, dy)
        p = f"c{ci}_"
        out[p + "dims"] = np.array([L, H, I, B, T, seed], np.int64)
        for l in range(L):
            out[p + f"w{l}"] = w[l]
            out[p + f"r{l}"] = r[l]
            out[p + f"b{l}"] = b[l]
            if state:
                out[p + f"h0_{l}"] = h0[l]
                out[p + f"c0_{l}"] = c0[l]
        out[p + "x"] = x
        out[p + "dy"] = dy
        for k, v in res.items():
            if isinstance(v, list):
                for l, a in enumerate(v):
                    out[p + f"{k}{l}"] = a
            else:
                out[p + k] = v
    path = os.path.join(HERE, "lstm_golden.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path), "bytes,", len(CASES), "cases")


if __name__ == "__main__":
    main()
