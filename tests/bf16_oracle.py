"""bf16 storage-point emulation of the float64 oracle (test infrastructure).

The device's bf16 path stores features, aggregates and activations h_k in
bf16, and on the tensor-core path its GEMM operands (weights, dz, dlogits)
are bf16 too; arithmetic accumulates in fp32.  These helpers run the float64
oracle (oracle/model.py, restating model.py:213-287) with the same values
rounded to bf16 at the same points, so the remaining device/oracle gap is
fp32-vs-f64 accumulation plus the occasional one-ulp rounding difference.
"""
import numpy as np
import torch

from oracle import kernels as OK
from oracle import model as OM
from oracle.sampler import sample_micrograph as o_sample, stream_key


def _bf(a):
    """float64 -> float32 -> bf16 (round to nearest even) -> float64, in numpy
    (no torch: the helpers also run in forked pool workers)."""
    x = np.ascontiguousarray(np.asarray(a, np.float64).astype(np.float32))
    u = x.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def forward_bf16(m, x_rows, P, tc=False):
    """OM.forward with the bf16 storage points of the device path emulated:
    features, every aggregate and every activation h_k are rounded to bf16;
    on the tensor-core path the layer weights are bf16 operands too."""
    need, steps = OM.build_plan(m)
    x = _bf(x_rows)
    h = [x[np.searchsorted(m.vertices, need[0])]]
    aggs, zs = [], []
    for k, (self_pos, dpos, spos, deg) in enumerate(steps, start=1):
        prev = h[-1]
        s = np.zeros((len(need[k]), prev.shape[1]))
        np.add.at(s, dpos, prev[spos])
        own = prev[self_pos]
        if P.arch == OM.GCN:
            agg = (s + own) / (deg + 1.0)[:, None]
        else:
            has = (deg > 0)[:, None]
            agg = np.concatenate([own, np.where(has, s / np.maximum(deg, 1.0)[:, None], own)], 1)
        agg = _bf(agg)
        z = agg @ (_bf(P.W[k - 1]) if tc else P.W[k - 1]) + P.b[k - 1]
        aggs.append(agg)
        zs.append(z)
        h.append(_bf(np.maximum(z, 0.0)))
    return dict(need=need, steps=steps, h=h, aggs=aggs, zs=zs,
                logits=h[-1][0] @ (_bf(P.Wc) if tc else P.Wc))


def grads_bf16(st, label, P, tc, masks=None):
    """OM.loss_and_grads; on the tensor-core path dW_k = agg_kᵀ bf16(dz_k).
    masks: optional per-layer ReLU masks (need[k] x H booleans) to use instead
    of z_k > 0 -- the device's own masks, so a pre-activation that lands on the
    other side of 0 after a one-ulp bf16 difference upstream does not flip a
    whole gradient term (the 'mask-forced' comparison)."""
    if not tc:
        if masks is None:
            return OM.loss_and_grads(st, label, P)
        st = dict(st, zs=[np.where(m, 1.0, -1.0) for m in masks])
        return OM.loss_and_grads(st, label, P)
    orig = [w.copy() for w in P.W]
    # run the exact backward, then redo the weight gradients with bf16 dz
    loss, G = OM.loss_and_grads(st, label, P)
    lg = st["logits"]
    e = np.exp(lg - lg.max())
    dl = e / e.sum()
    dl[label] -= 1.0
    L = len(P.W)
    # tensor-core head: bf16 dlogits and bf16 W_c operands
    G.Wc[...] = np.outer(st["h"][L][0], _bf(dl))
    dh = np.zeros_like(st["h"][L])
    dh[0] = _bf(P.Wc) @ _bf(dl)
    for k in range(L, 0, -1):
        self_pos, dpos, spos, deg = st["steps"][k - 1]
        dz = dh * (masks[k - 1] if masks is not None else (st["zs"][k - 1] > 0.0))
        G.W[k - 1][...] = st["aggs"][k - 1].T @ _bf(dz)
        G.b[k - 1][...] = dz.sum(0)  # from the bf16 chain too (dh = bf16 W_c @ bf16 dl, ...)
        # tensor-core dX (layers >= 2): bf16 dz times bf16 W
        dagg = _bf(dz) @ _bf(orig[k - 1]).T if orig[k - 1].shape[0] % 64 == 0 else dz @ orig[k - 1].T
        prev = np.zeros_like(st["h"][k - 1])
        if P.arch == OM.GCN:
            part = dagg / (deg + 1.0)[:, None]
            prev[self_pos] += part
            np.add.at(prev, spos, part[dpos])
        else:
            w = st["h"][k - 1].shape[1]
            has = deg > 0
            prev[self_pos] += dagg[:, :w]
            np.add.at(prev, spos, np.where(has[:, None], dagg[:, w:] / np.maximum(deg, 1.0)[:, None], 0.0)[dpos])
            prev[self_pos] += np.where(has[:, None], 0.0, dagg[:, w:])
        dh = prev
    return loss, G


def oracle_cell(off, tgt, roots, fo, sseed, it_key, P, D, fstate, lseed, C, bf16_feats=False,
                tc=False, micros=None, masks=None):
    """Oracle gradients; with bf16_feats the oracle rounds features, aggregates and
    activations to bf16 where the device stores them (arithmetic stays float64).
    micros: pre-sampled micrographs (one per root), else sampled from (off, tgt)."""
    G = P.zeros()
    losses = []
    for i, r in enumerate(roots.tolist()):
        m = micros[i] if micros is not None else o_sample(
            off, tgt, r, fo, stream_key(sseed, *it_key, r), draw=OK.sample_frontier_nb)
        x = OK.feature_rows(m.vertices, D, fstate)
        st = forward_bf16(m, x, P, tc) if bf16_feats else OM.forward(m, x, P)
        lab = int(OM.labels([r], C, lseed)[0])
        mk = masks[i] if masks is not None else None
        loss, g = (grads_bf16(st, lab, P, tc, mk) if bf16_feats
                   else OM.loss_and_grads(st, lab, P))
        OM.add_into(G, g)
        losses.append(loss)
    return np.array(losses), G


def errors(got, want):
    """(max-abs error / max|ref|, norm-relative error) of one tensor."""
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    scale = max(np.abs(want).max(), 1e-30)
    return (float(np.abs(got - want).max() / scale),
            float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30)))


def _cell_chunk(args):
    micros, roots, P, D, fstate, lseed, C, tc = args
    return oracle_cell(None, None, roots, None, None, None, P, D, fstate, lseed, C,
                       bf16_feats=True, tc=tc, micros=micros)


def oracle_cell_parallel(pool, micros, roots, P, D, fstate, lseed, C, tc=True, parts=16):
    """oracle_cell (bf16 storage points) with the roots split over a process pool;
    per-root losses in root order and the summed gradients."""
    idx = np.array_split(np.arange(len(roots)), parts)
    jobs = [([micros[i] for i in ix], roots[ix], P, D, fstate, lseed, C, tc) for ix in idx if len(ix)]
    res = pool.map(_cell_chunk, jobs)
    G = P.zeros()
    for _, g in res:
        OM.add_into(G, g)
    return np.concatenate([l for l, _ in res]), G
