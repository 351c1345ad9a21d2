"""TEST INFRASTRUCTURE ONLY — native-mode parity accounting.

The reference's Index + Tables phases (adc.py:140-174) recomputed on the
host for a sample of queries, with the rotation done by the reference's own
call — `(v @ pq.rotation.T).astype(np.float32)` (adc.py:108-111), i.e. this
host's numpy / OpenBLAS sgemv — and everything else by the pinned oracle
(probe ivf.py:166-182, compute_tables adc.py:61-75, find_qmax
qadc.py:157-194, qmin adc.py:173, quantize_tables qadc.py:124-147).
`account` compares the GPU's intermediates (DeviceIndex.tables) with them:
fp32 LUT bit mismatches and relative error, uint8 bucket flips, qmax
mismatches, probe-order mismatches.

Imported only by tests/ and bench.py's parity leg (the checker), never by
the product package.
"""

from __future__ import annotations

import numpy as np

from oracle import oracle as orc


def reference_rotate(rotation, v):
    """adc.py:108-111 exactly as the reference runs it (1-D v -> sgemv)."""
    if rotation is None:
        return np.asarray(v, np.float32)
    return (np.asarray(v, np.float32) @ rotation.T).astype(np.float32)


def reference_tables(queries, codebooks, rotation, coarse, ma, flat, R, init, cells=None):
    """Per query: probe order, fp32 LUTs, qmax, uint8 LUTs, fp32 qmin/delta
    of the reference on this host. `flat` = the oracle's (blocks, blk_off,
    ids, count) layout (only the first probed list of each query is read).
    `cells` (Q, ma) may be passed to skip the probe (then only the tables
    are recomputed)."""
    blocks, blk_off, _, count = flat
    q = np.ascontiguousarray(queries, np.float32)
    cb = np.ascontiguousarray(codebooks, np.float32)
    m = cb.shape[0]
    nq = q.shape[0]
    slots = ma if coarse is not None else 1
    mrows = m // 2
    out = {"cells": np.zeros((nq, slots), np.int64),
           "lut": np.empty((nq, slots, m, 16), np.float32),
           "qmax": np.empty(nq, np.float32),
           "qt": np.empty((nq, slots, m, 16), np.uint8),
           "qmin": np.empty((nq, slots), np.float32),
           "delta": np.empty((nq, slots), np.float32)}
    for i in range(nq):
        if coarse is None:
            cl, res = np.zeros(1, np.int64), q[i][None, :]
        elif cells is not None:
            cl = np.asarray(cells[i], np.int64)
            res = (q[i][None, :] - coarse[cl]).astype(np.float32)
        else:
            cl, res = orc.probe(coarse, q[i], ma)
        out["cells"][i] = cl
        qmax = None
        for s in range(slots):
            tab = orc.compute_tables(cb, reference_rotate(rotation, res[s]))
            out["lut"][i, s] = tab
            if qmax is None:
                c = int(cl[0])
                b0, b1 = int(blk_off[c]), int(blk_off[c + 1])
                lst = blocks[b0 * mrows * 16:b1 * mrows * 16].reshape(-1, mrows, 16)
                qmax = orc.find_qmax(tab, lst, int(count[c]), R, init)
                out["qmax"][i] = np.float32(qmax)
            qmin = min(float(tab.min()), qmax)
            qt, delta = orc.quantize_tables(tab, qmin, qmax)
            out["qt"][i, s] = qt
            out["qmin"][i, s] = np.float32(qmin)
            out["delta"][i, s] = np.float32(delta)
    return out


def account(gpu: dict, ref: dict) -> dict:
    """Native-mode divergence counts of the GPU's tables vs the reference's
    (both dicts of numpy arrays with the keys of reference_tables)."""
    g_lut, r_lut = gpu["lut"], ref["lut"]
    lut_diff = g_lut.view(np.uint32) != r_lut.view(np.uint32)
    # relative error with an absolute floor of 1e-6 * max|LUT| per table
    # set (documented choice for near-zero entries)
    floor = 1e-6 * np.abs(r_lut).max(axis=(2, 3), keepdims=True)
    rel = np.abs(g_lut.astype(np.float64) - r_lut) / np.maximum(np.abs(r_lut), floor)
    flips = gpu["qt"] != ref["qt"]
    qmax_mis = gpu["qmax"].view(np.uint32) != ref["qmax"].view(np.uint32)
    cells_mis = (gpu["cells"] != ref["cells"]).any(axis=1)
    flip_q = flips.any(axis=(1, 2, 3)) | qmax_mis | cells_mis
    return {
        "queries": int(g_lut.shape[0]),
        "cells_mismatch_queries": int(cells_mis.sum()),
        "lut_entries": int(lut_diff.size),
        "lut_bits_mismatch": int(lut_diff.sum()),
        "lut_max_rel_err": float(rel.max()) if rel.size else 0.0,
        "qmax_mismatch": int(qmax_mis.sum()),
        "u8_flips": int(flips.sum()),
        "u8_flip_queries": int(flips.any(axis=(1, 2, 3)).sum()),
        "queries_with_any_divergence": int(flip_q.sum()),
        "_diverged": flip_q,
    }


def compare_results(gi, gd, ri, rd, diverged=None) -> dict:
    """Per-query top-R comparison: ids exact, fp32 distance bits exact;
    with `diverged` (bool per query), also the counts over the queries
    whose tables did not diverge."""
    gi, ri = np.asarray(gi), np.asarray(ri)
    gd = np.ascontiguousarray(gd, np.float32).view(np.uint32)
    rd = np.ascontiguousarray(rd, np.float32).view(np.uint32)
    ids_ok = np.array([np.array_equal(gi[i], ri[i]) for i in range(gi.shape[0])])
    d_ok = np.array([np.array_equal(gd[i], rd[i]) for i in range(gi.shape[0])])
    out = {"queries": int(gi.shape[0]), "ids_exact": int(ids_ok.sum()),
           "dist_bits_exact": int((ids_ok & d_ok).sum())}
    if diverged is not None:
        clean = ~np.asarray(diverged)
        out["clean_queries"] = int(clean.sum())
        out["clean_exact"] = int((ids_ok & d_ok & clean).sum())
    return out
