"""GPU diagnostics: run parity cases one per subprocess (bounded by a timeout) and print
per-tensor errors, the chosen schedule and wall time. Not a pytest module.

  python tests/gpu_diag.py [case-filter]
"""
import json
import os
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

CASES = [
    # (L, H, I, B, T, precision, schedule, mode)
    (2, 64, 64, 16, 8, "bf16", "persistent", "both-debug"),
    (3, 96, 40, 20, 10, "bf16", "persistent", "both-debug"),
    (2, 130, 70, 33, 5, "bf16", "persistent", "both-debug"),
    (2, 130, 70, 33, 5, "fp32", "persistent", "both-debug"),
    (4, 512, 512, 64, 100, "bf16", "persistent", "both"),
    (4, 512, 512, 64, 100, "fp32", "auto", "both"),
    (4, 512, 512, 64, 100, "bf16", "stepwise", "both"),
    (4, 1024, 1024, 16, 200, "bf16", "auto", "both"),
    (4, 2048, 2048, 64, 100, "bf16", "auto", "both"),
]


def child(spec):
    L, H, I, B, T, prec, sched, mode = spec
    sys.path.insert(0, ROOT)
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import oracle
    from paper_1604_01946_b200 import Engine
    from parity import compare, errors, make_case, run_device
    d = oracle.Dims(L, H, I, B, T)
    c, params, x, dy, h0, c0 = make_case(d, seed=7, bias=True, state=True)
    try:
        ref = oracle.Reference()
    except Exception:
        ref = oracle.Restatement()
    w = [p.w for p in params]
    r = [p.r for p in params]
    b = [np.ascontiguousarray(p.bias) for p in params]
    t0 = time.time()
    eng = Engine(c, precision=prec, schedule=sched)
    out = {"describe": eng.describe()}
    if mode == "fwd":
        fwd = eng.forward(params, x, True, h0, c0)
        ro = ref.run(c, w, r, b, x, h0, c0, None)
        out["y"] = errors(fwd.y, ro["y"])
        for l in range(L):
            out[f"h{l}"] = errors(fwd.tape.h_seq[l], ro["h_seq"][l])
            out[f"g{l}"] = errors(fwd.tape.gates_seq[l], ro["gates_seq"][l])
    else:
        dev = run_device(eng, params, x, dy, h0, c0)
        ro = ref.run(c, w, r, b, x, h0, c0, dy)
        out["rows"] = [(n, round(a, 9), round(m, 9)) for n, a, m in compare(dev, ro, c)]
    out["sec"] = round(time.time() - t0, 2)
    print("RESULT " + json.dumps(out), flush=True)


def main():
    filt = sys.argv[1] if len(sys.argv) > 1 else ""
    for spec in CASES:
        env = dict(os.environ, RW_FLAG_TIMEOUT_MS="4000")
        name = "L{}H{}I{}B{}T{}-{}-{}-{}".format(*spec)
        if filt not in name:
            continue
        if spec[-1].endswith("-debug"):
            env["RW_DEBUG_HANG_S"] = "15"
        if spec[-1].endswith("-onesm"):
            env["RW_MIN_SMEM_KB"] = "120"
        spec = list(spec[:-1]) + [spec[-1].split("-")[0]]
        t0 = time.time()
        try:
            p = subprocess.run([sys.executable, __file__, "--child", json.dumps(spec)], env=env,
                               capture_output=True, text=True, timeout=240)
            res = [l for l in p.stdout.splitlines() if l.startswith("RESULT ")]
            msg = res[0][7:] if res else ("rc=%d %s" % (p.returncode, (p.stderr or p.stdout)[-1500:]))
        except subprocess.TimeoutExpired:
            msg = "TIMEOUT (240 s)"
        print(f"=== {name} [{time.time() - t0:.1f}s]\n{msg}", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--child":
        child(json.loads(sys.argv[2]))
    else:
        main()
