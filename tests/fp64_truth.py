"""fp64 ground truth of the LSTM forward + backward on the GPU (torch, test infrastructure only):
the reference's arithmetic (cells.hpp:227-260 forward, 402-449 backward; engine.hpp:178-217
weight gradients) evaluated in float64. Used by tests/test_parity_full.py to decide whether a
fp32-parity difference from the reference CPU engine is our error or the reference's own fp32
rounding: at config E (K = B*T = 25600 long gradient sums) the reference itself sits ~1e-5 from
the truth, so there the contract is "at least as close to the fp64 truth as the reference is".
Matrices follow the reference layout (column-major, column t*B + b)."""
import numpy as np
import torch


def _t(a, dev):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64).T)).to(dev)  # (cols, rows)


def lstm_truth(c, params, x, dy, h0=None, c0=None, device="cuda"):
    """-> dict like oracle.Reference.run (float64 numpy, reference layouts): y, dx0, dh0, dc0,
    dw, dr, db and h_seq / c_seq final blocks (hT, cT)."""
    L, H, B, T = c.layers, c.hidden, c.batch, c.steps
    dev = torch.device(device)
    W = [torch.from_numpy(np.asarray(p.w, np.float64)).to(dev) for p in params]   # (4H, I_l)
    R = [torch.from_numpy(np.asarray(p.r, np.float64)).to(dev) for p in params]   # (4H, H)
    bias = [torch.from_numpy(np.asarray(p.bias, np.float64)).to(dev) for p in params]
    X = _t(x, dev)  # (B T, I)
    DY = _t(dy, dev)  # (B T, H)
    hs, cs, gs, tcs = [], [], [], []
    inp = X
    for l in range(L):
        h = _t(h0[l], dev) if h0 is not None else torch.zeros(B, H, dtype=torch.float64, device=dev)
        cc = _t(c0[l], dev) if c0 is not None else torch.zeros(B, H, dtype=torch.float64, device=dev)
        zx = inp @ W[l].T  # (B T, 4H): W.x for every step
        hseq = [h]
        cseq = [cc]
        gseq, tseq = [], []
        for t in range(T):
            a = (zx[t * B:(t + 1) * B] + h @ R[l].T) + bias[l]
            i = torch.sigmoid(a[:, :H])
            f = torch.sigmoid(a[:, H:2 * H])
            o = torch.sigmoid(a[:, 2 * H:3 * H])
            cb = torch.tanh(a[:, 3 * H:])
            cc = f * cc + i * cb
            tc = torch.tanh(cc)
            h = o * tc
            hseq.append(h)
            cseq.append(cc)
            gseq.append(torch.cat([i, f, o, cb], 1))
            tseq.append(tc)
        hs.append(torch.stack(hseq))   # (T+1, B, H)
        cs.append(torch.stack(cseq))
        gs.append(torch.stack(gseq))   # (T, B, 4H)
        tcs.append(torch.stack(tseq))
        inp = hs[-1][1:].reshape(T * B, H)
        del zx
    out = {"y": hs[-1][1:].reshape(T * B, H).T.cpu().numpy(),
           "hT": [hs[l][T].T.cpu().numpy() for l in range(L)],
           "cT": [cs[l][T].T.cpu().numpy() for l in range(L)]}
    dabove = DY.reshape(T, B, H)
    dw, dr, db, dh0, dc0 = [None] * L, [None] * L, [None] * L, [None] * L, [None] * L
    dx0 = None
    for l in range(L - 1, -1, -1):
        carry_h = torch.zeros(B, H, dtype=torch.float64, device=dev)
        carry_c = torch.zeros(B, H, dtype=torch.float64, device=dev)
        dG = torch.empty(T, B, 4 * H, dtype=torch.float64, device=dev)
        for t in range(T - 1, -1, -1):
            g = gs[l][t]
            i, f, o, cb = g[:, :H], g[:, H:2 * H], g[:, 2 * H:3 * H], g[:, 3 * H:]
            tc = tcs[l][t]
            cp = cs[l][t]  # c_{t-1}
            dh = dabove[t] + carry_h
            dc = carry_c + dh * o * (1 - tc * tc)
            gi = dc * cb * i * (1 - i)
            gf = dc * cp * f * (1 - f)
            go = dh * tc * o * (1 - o)
            gc = dc * i * (1 - cb * cb)
            carry_c = dc * f
            dGt = torch.cat([gi, gf, go, gc], 1)
            dG[t] = dGt
            carry_h = dGt @ R[l]  # R^T dG for step t-1
        dh0[l] = carry_h.T.cpu().numpy()
        dc0[l] = carry_c.T.cpu().numpy()
        G2 = dG.reshape(T * B, 4 * H)
        linp = X if l == 0 else hs[l - 1][1:].reshape(T * B, H)
        dw[l] = (G2.T @ linp).cpu().numpy()
        dr[l] = (G2.T @ hs[l][:T].reshape(T * B, H)).cpu().numpy()
        db[l] = G2.sum(0).cpu().numpy()
        d = G2 @ W[l]  # (B T, I_l): d_above of the layer below, or dx0
        if l == 0:
            dx0 = d.T.cpu().numpy()
        else:
            dabove = d.reshape(T, B, H)
        del dG, G2
    out.update(dx0=dx0, dh0=dh0, dc0=dc0, dw=dw, dr=dr, db=db)
    return out
