"""Whole-network float twin of the integer model (NEXT-2; TEST INFRASTRUCTURE ONLY).

The paper's motivation (Fig. 2b/c): "non-deterministic floating-point
inference leads to cross-platform decoding failure" — an entropy decoder fed a CDF that
differs from the encoder's in one entry decodes garbage from there on, and the decoded
cloud "collapses"; the integer-only pipeline decodes bit-exactly everywhere.

The twin is the SAME network as the integer model (inputs.Model), dequantised: every
layer computes acc = W x + b in float32 with the int8 weights as floats, then y =
acc * s with s = m_pos / 2^r (acc >= 0) or m_neg / 2^r (the requant multiplier of Eq.14
without its rounding and clipping; the fused PReLU of reading Q18).  The wiring is the
oracle's O7 step by step (Eq.4-11, readings Q2-Q9, Q14): shallow ResBlock + Up/Prune,
deep embedding + K2S2 down chain + XFP ResBlock + up chain, Eq.7 predictor.  Logits in
nats (z * m_l / 2^r_l / 256, reading Q20), a float32 softmax, and reading Q21's
cumulative floors give the Q16 pmf that drives a one-lane rANS (reading O9).

A twin runs on a backend: numpy float32 ("cpu") or torch float32 on cuda:0 ("cuda",
TF32 off), and in an evaluation order: "fused" (each conv as one matmul over the 27
gathered offsets) or "per_offset" (the offsets accumulated one matmul at a time, last
offset first).  The octree and kernel maps are integer (the oracle's).
"""
from __future__ import annotations

import numpy as np

from oracle import oracle as O

M = 1 << 16
NC = 255


def quantise_pmf(logits: np.ndarray) -> np.ndarray:
    """Float32 softmax, then reading Q21's cumulative floors: C_i = i + floor(E_i 65281 / E_255)."""
    l = np.asarray(logits, np.float32)
    e = np.exp(l - l.max(1, keepdims=True)).astype(np.float32)
    E = np.cumsum(e, 1, dtype=np.float32)
    frac = (E / E[:, -1:]).astype(np.float32)
    C = np.arange(1, NC + 1)[None, :] + np.floor(frac.astype(np.float64) * 65281).astype(np.int64)
    C[:, -1] = M
    C = np.concatenate([np.zeros((len(C), 1), np.int64), C], 1)
    p = np.diff(C, axis=1)
    assert (p >= 1).all() and (p.sum(1) == M).all()
    return p


def rans_encode(sym, pmfs):
    """Reading O9, one lane: returns (words, final state); sym in 0..254."""
    cum = np.concatenate([np.zeros((len(pmfs), 1), np.int64), np.cumsum(pmfs, 1)], 1)
    x, words = 1 << 16, []
    for i in reversed(range(len(sym))):
        s = int(sym[i])
        f, c = int(pmfs[i, s]), int(cum[i, s])
        if x >= f << 16:
            words.append(x & 0xFFFF)
            x >>= 16
        x = ((x // f) << 16) + (x % f) + c
    return words[::-1], x


def rans_decode(words, x, pmfs, pos=0):
    """Decode len(pmfs) symbols; returns (symbols 0..254, next word position, state)."""
    cum = np.concatenate([np.zeros((len(pmfs), 1), np.int64), np.cumsum(pmfs, 1)], 1)
    out = np.zeros(len(pmfs), np.int64)
    for i in range(len(pmfs)):
        slot = x & 0xFFFF
        s = min(max(int(np.searchsorted(cum[i], slot, side="right") - 1), 0), NC - 1)
        out[i] = s
        x = int(pmfs[i, s]) * (x >> 16) + slot - int(cum[i, s])
        if x < (1 << 16):
            x = (x << 16) | (words[pos] if pos < len(words) else 0)
            pos += 1
    return out, pos, x


class FloatTwin:
    """Float32 forward pass of the integer model's network on one backend / order."""

    def __init__(self, model, backend: str = "cpu", order: str = "fused"):
        self.m, self.backend, self.order = model, backend, order
        self.C = model.C
        if backend == "cuda":
            import torch
            torch.backends.cuda.matmul.allow_tf32 = False
            self.torch = torch

    # ---- backend primitives (float32) ----
    def arr(self, a):
        a = np.asarray(a, np.float32)
        return self.torch.from_numpy(a).cuda() if self.backend == "cuda" else a

    def host(self, a):
        return a.cpu().numpy() if self.backend == "cuda" else a

    def mm(self, x, W):  # x [n, k] @ W[o, k]^T
        return x @ W.T

    def scale(self, acc, rq):
        sp, sn = np.float32(rq.m_pos / 2.0 ** rq.r), np.float32(rq.m_neg / 2.0 ** rq.r)
        if self.backend == "cuda":
            return self.torch.where(acc >= 0, acc * float(sp), acc * float(sn))
        return np.where(acc >= 0, acc * sp, acc * sn).astype(np.float32)

    def gather(self, x, idx):  # rows x[idx], idx -1 -> zero row
        n = x.shape[0]
        if self.backend == "cuda":
            z = self.torch.cat([x, self.torch.zeros((1, x.shape[1]), dtype=x.dtype, device=x.device)])
            ii = self.torch.from_numpy(np.where(idx < 0, n, idx).astype(np.int64)).cuda()
            return z[ii]
        z = np.concatenate([x, np.zeros((1, x.shape[1]), np.float32)])
        return z[np.where(idx < 0, n, idx)]

    def cat(self, xs, axis=1):
        return self.torch.cat(xs, axis) if self.backend == "cuda" else np.concatenate(xs, axis)

    # ---- layers ----
    def conv3(self, x, nbr, W):
        """sum_delta W_delta x[nbr(., delta)]; W int8 [27][out][in]."""
        Wf = np.asarray(W, np.float32)
        if self.order == "fused":
            g = self.gather(x, nbr.reshape(-1)).reshape(nbr.shape[0], 27 * x.shape[1])
            Wcat = self.arr(Wf.transpose(1, 0, 2).reshape(Wf.shape[1], 27 * Wf.shape[2]))
            return self.mm(g, Wcat)
        acc = None
        for dl in reversed(range(27)):
            t = self.mm(self.gather(x, nbr[:, dl]), self.arr(Wf[dl]))
            acc = t if acc is None else acc + t
        return acc

    def resblock_cc(self, F, nbr, Wa, ba, rqa, Wb, bb, k_s, rqb):
        h = self.scale(self.conv3(F, nbr, Wa) + self.arr(ba), rqa)
        return self.scale(self.conv3(h, nbr, Wb) + F * float(k_s) + self.arr(bb), rqb)

    def up_prune(self, u, S, X):
        C = self.C
        oh = np.zeros((len(X), NC), np.float32)
        oh[np.arange(len(X)), X.astype(np.int64) - 1] = u.q_one
        x = self.cat([S, self.arr(oh)])
        U = self.scale(self.mm(x, self.arr(u.W)) + self.arr(u.b), u.rq)
        rows = [(p * 8 + c) for p in range(len(X)) for c in range(8) if (int(X[p]) >> c) & 1]
        U = U.reshape(len(X) * 8, C)
        ii = np.array(rows, np.int64)
        return U[self.torch.from_numpy(ii).cuda()] if self.backend == "cuda" else U[ii]

    def down(self, dn, g, child_keys, parent_keys):
        C = self.C
        par = np.searchsorted(parent_keys, child_keys >> np.uint64(3))
        cidx = (child_keys & np.uint64(7)).astype(np.int64)
        Wf = np.asarray(dn.W, np.float32)  # [8][out][in]
        # every child row through its child-index matrix, then summed into its parent
        Wsel = self.arr(Wf)
        if self.backend == "cuda":
            t = self.torch
            ci = t.from_numpy(cidx).cuda()
            y = t.einsum("noi,ni->no", Wsel[ci], g)
            acc = t.zeros((len(parent_keys), C), dtype=y.dtype, device=y.device)
            acc.index_add_(0, t.from_numpy(par.astype(np.int64)).cuda(), y)
        else:
            y = np.einsum("noi,ni->no", Wf[cidx], g).astype(np.float32)
            acc = np.zeros((len(parent_keys), C), np.float32)
            order = range(len(par)) if self.order == "fused" else reversed(range(len(par)))
            for j in order:
                acc[par[j]] += y[j]
        return self.scale(acc + self.arr(dn.b), dn.rq)

    def head_pmf(self, hd, F):
        a = self.scale(self.mm(F, self.arr(hd.W1)) + self.arr(hd.b1), hd.rq1)
        z = self.mm(a, self.arr(hd.W2)) + self.arr(hd.b2)
        lg = self.host(z).astype(np.float32) * np.float32(hd.rq_logit.m_pos / 2.0 ** hd.rq_logit.r / 256.0)
        return quantise_pmf(lg)

    # ---- the level-wise network (oracle O7) ----
    def reset(self):
        self.F_prev = None
        self.F_D = None

    def level_pmf(self, keys, codes, d, L):
        m, C = self.m, self.C
        D = L - 1 - m.n_deep
        if d <= D:
            s = m.shallow[d]
            if d == m.R:
                self.F_prev = self.arr(m.E0[codes[d - 1].astype(np.int64) - 1])
            nbr = O.kernel_map(keys[d - 1], d - 1)
            S = self.resblock_cc(self.F_prev, nbr, s.Wa, s.ba, s.rqa, s.Wb, s.bb, s.k_s, s.rqb)
            Fd = self.up_prune(s.up, S, codes[d - 1])
            self.F_prev = Fd
            if d == D:
                self.F_D = Fd
            return self.head_pmf(s.head, Fd)
        j = d - D
        dp = m.deep[j - 1]
        g = self.arr(dp.E[codes[d - 1].astype(np.int64) - 1])
        for s_ in range(j - 1):
            k = d - 1 - s_
            g = self.down(dp.downs[s_], g, keys[k], keys[k - 1])
        nbr = O.kernel_map(keys[D], D)
        if m.flags & 1:  # XFP off
            H = self.resblock_cc(g, nbr, dp.Wa, dp.ba, dp.rqa, dp.Wb, dp.bb, dp.k_s, dp.rqb)
        else:
            x = self.cat([self.F_D, g])
            h = self.scale(self.conv3(x, nbr, dp.Wa) + self.arr(dp.ba), dp.rqa)
            H = self.scale(self.conv3(h, nbr, dp.Wb) + self.mm(x, self.arr(dp.P)) + self.arr(dp.bb), dp.rqb)
        cur = H
        for k in range(D, d):
            cur = self.up_prune(dp.ups[k - D], cur, codes[k])
        return self.head_pmf(dp.head, cur)


def float_encode(twin: FloatTwin, pts, L):
    """Encode with the float twin: per level one rANS lane over the twin's pmfs."""
    keys, codes = O.build_octree(pts, L)
    twin.reset()
    levels, pmfs = [], []
    for d in range(twin.m.R, L):
        p = twin.level_pmf(keys, codes, d, L)
        pmfs.append(p)
        levels.append(rans_encode(codes[d].astype(np.int64) - 1, p))
    return {"raw": [codes[d] for d in range(twin.m.R)], "levels": levels, "n_leaf": keys[L].size}, pmfs


def float_decode(twin: FloatTwin, stream, L, max_growth=4.0):
    """Level-serial decode with the float twin (Eq.2).  Stops expanding when a level grows
    beyond max_growth x the encoded leaf count (a collapsed decode).  Returns (keys at the
    last decoded depth, depth reached, per-level pmfs)."""
    R = twin.m.R
    keys = [np.array([0], np.uint64)]
    codes = []
    for d in range(R):
        codes.append(stream["raw"][d])
        keys.append(O.expand(keys[d], codes[d]))
    twin.reset()
    pmfs = []
    for d in range(R, L):
        p = twin.level_pmf(keys, codes, d, L)
        pmfs.append(p)
        words, x = stream["levels"][d - R]
        # the encoder's final state starts the decoder (reading O9)
        sym, _, _ = rans_decode(words, x, p)
        codes.append((sym + 1).astype(np.uint8))
        keys.append(O.expand(keys[d], codes[d]))
        if keys[-1].size > max_growth * stream["n_leaf"]:
            return keys[-1], d + 1, pmfs
    return keys[L], L, pmfs
