"""Parity margin probe (GPU box): max errors per config against the fp64
oracle, plus the structure of the gradient error of the worst case.

    python tools/parity_probe.py [--only NAME ...] [--json out.json]

For each config prints max |rel cost err|, max |grad err| and where the
gradient error sits (blank column vs label columns). For the analysis it
recovers the occupancies from the gradients (occ = softmax - grad, softmax
from the fp64 logits) and splits the relative occupancy error into the part
common to a frame (a per-frame scale, what a per-frame renormalisation
would remove) and the rest.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (test infrastructure: the checker)
from paper_1512_02595_b200 import ctc as dctc  # noqa: E402
from paper_1512_02595_b200.synth import fixed_shape_batch, make_batch, sortagrad_lengths  # noqa: E402


def configs():
    out = {}
    out["english"] = lambda: fixed_shape_batch(29, 700, 150, 64, seed=1234)
    out["english-peaked8"] = lambda: fixed_shape_batch(29, 700, 150, 16, seed=77, scale=8.0)
    out["t1500-peaked8"] = lambda: fixed_shape_batch(29, 1500, 300, 16, seed=78, scale=8.0)
    out["t1500-flat"] = lambda: fixed_shape_batch(29, 1500, 300, 16, seed=79)
    out["mandarin-b64"] = lambda: fixed_shape_batch(6000, 350, 60, 64, seed=1234)

    def sorta(n, seed):
        T, L = sortagrad_lengths(n, seed=seed)
        o = np.argsort(T, kind="stable")
        return make_batch(29, T[o], L[o], seed=6)

    out["sortagrad-512"] = lambda: sorta(512, 7)
    out["sortagrad-320"] = lambda: sorta(320, 13)

    def blank0():
        acts, flat, ll, il = fixed_shape_batch(29, 700, 150, 16, seed=31)
        flat = flat + 1  # labels in 1..28, blank = 0
        return acts, flat.astype(np.int32), ll, il

    out["blank0"] = blank0
    return out


def softmax64(acts):
    x = acts.astype(np.float64)
    m = x.max(axis=2, keepdims=True)
    e = np.exp(x - m)
    return e / e.sum(axis=2, keepdims=True)


def analyse(acts, il, g, rg, blank):
    sm = softmax64(acts)
    occ_g = sm - g.astype(np.float64)
    occ_r = sm - rg
    T, B, A = acts.shape
    common, resid, blank_err, label_err = [], [], 0.0, 0.0
    lab = np.ones(A, bool)
    lab[blank] = False
    norm_abs, norm_where = 0.0, None
    for b in range(B):
        for t in range(int(il[b])):
            r = occ_r[t, b]
            gg = occ_g[t, b]
            m = r > 1e-2
            if m.sum() >= 2:
                rel = (gg[m] - r[m]) / r[m]
                c = float(np.sum(rel * r[m]) / np.sum(r[m]))  # mass-weighted common scale
                common.append(abs(c))
                resid.append(float(np.max(np.abs(rel - c))))
            # what a per-frame renormalisation would leave on the label columns:
            # remove the frame's common scale (estimated on label cells with mass)
            ml = lab & (r > 1e-3)
            if ml.any():
                c = float(np.sum((gg[ml] - r[ml])) / np.sum(r[ml]))
                e = np.abs(gg[lab] / (1.0 + c) - r[lab])
                k = int(np.argmax(e))
                if e[k] > norm_abs:
                    norm_abs = float(e[k])
                    norm_where = (b, t, int(np.arange(A)[lab][k]), float(r[lab][k]), float(gg[lab][k]), c)
    err = np.abs(g.astype(np.float64) - rg)
    blank_err = float(err[:, :, blank].max())
    mask = np.ones(A, bool)
    mask[blank] = False
    label_err = float(err[:, :, mask].max())
    return {"frame_common_rel_max": max(common) if common else 0.0,
            "frame_common_rel_mean": float(np.mean(common)) if common else 0.0,
            "within_frame_rel_max": max(resid) if resid else 0.0,
            "within_frame_rel_mean": float(np.mean(resid)) if resid else 0.0,
            "grad_err_blank_col": blank_err, "grad_err_label_cols": label_err,
            "label_err_after_frame_norm": norm_abs, "label_err_after_frame_norm_at": norm_where}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*")
    ap.add_argument("--json")
    ap.add_argument("--analyse", nargs="*", default=["t1500-peaked8", "sortagrad-320", "english-peaked8",
                                                     "sortagrad-512"])
    args = ap.parse_args()
    import torch

    res = {}
    for name, mk in configs().items():
        if args.only and name not in args.only:
            continue
        acts, flat, ll, il = mk()
        blank = 0 if name == "blank0" else acts.shape[2] - 1
        x = torch.from_numpy(acts).cuda()
        t0 = time.time()
        c, g = dctc.compute_ctc_loss(x, flat, ll, il, blank=blank)
        torch.cuda.synchronize()
        c = c.cpu().numpy().astype(np.float64)
        g = g.cpu().numpy()
        rc, rg = oracle.oracle_batch(acts, flat, ll, il, blank=blank, nthreads=os.cpu_count() or 8)
        fin = np.isfinite(rc)
        rel = float((np.abs(c[fin] - rc[fin]) / np.abs(rc[fin])).max()) if fin.any() else 0.0
        gerr = float(np.abs(g.astype(np.float64) - rg).max())
        r = {"B": int(len(il)), "max_rel_cost": rel, "max_abs_grad": gerr,
             "inf_match": bool(np.array_equal(np.isfinite(c), fin)), "seconds": time.time() - t0}
        if name in args.analyse:
            r.update(analyse(acts, il, g, rg, blank))
        res[name] = r
        print(name, json.dumps(r), flush=True)
    if args.json:
        with open(args.json, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
