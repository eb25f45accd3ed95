#!/usr/bin/env python
"""Fit the B200 pipeline model and train the DNN judge on a variant sweep.

Input: the JSON written by scripts/sweep_variants.py on the GPU.  Output:
  machines/b200_engine.json   fitted PipelineModel constants
  machines/b200_ranker.npz    DNN judge trained on measured pairwise outcomes
  profiles/ranker_<tag>.json  evaluation: per-layer Kendall tau of each
                              ranking vs the measured order, top-1 regret
                              (time of the chosen variant / best - 1), all
                              leave-one-layer-out for the fitted model.

    python scripts/fit_ranker.py gpurun_out/sweep_r1.json --tag r1
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

import numpy as np
from scipy.optimize import minimize

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2006_02230_b200 import rank, variants, workloads  # noqa: E402

PARAMS = ["mma_fixed", "mma_per_n", "l2_bytes_per_cycle", "kblock_fixed", "cluster_kb", "tile_fixed"]
LAYERS = {L.idx: L for L in workloads.resnet50_v1_layers()}


def samples(doc):
    out = []
    for rec in doc["layers"]:
        L = LAYERS[rec["idx"]]
        for vid, r in rec["variants"].items():
            if not r["legal"]:
                continue
            v = variants.TileVariant(vid, r["bn"], r["bk"], r["cluster"], rec["mode"])
            out.append((rec["idx"], rec["mode"], L, v, r["ms"] * 1e-3, r["stats"]))
    return out


def fit(data, batch, x0=None):
    base = rank.PipelineModel()
    x0 = np.log([getattr(base, k) for k in PARAMS]) if x0 is None else x0

    def model_of(x):
        return rank.PipelineModel(**{k: float(math.exp(v)) for k, v in zip(PARAMS, x)})

    def loss(x):
        pm = model_of(x)
        e = [math.log(pm.predict_seconds(L, v, batch) / t) for _, _, L, v, t, _ in data]
        return float(np.mean(np.square(e)))

    res = minimize(loss, x0, method="Nelder-Mead", options={"maxiter": 4000, "xatol": 1e-4,
                                                            "fatol": 1e-7})
    return model_of(res.x), res


def evaluate(doc, batch, predict):
    """predict(layer_rec, vid) -> score (smaller = better)."""
    taus, regrets, dflt_regrets = [], [], []
    for rec in doc["layers"]:
        vs = {k: r for k, r in rec["variants"].items() if r["legal"]}
        if len(vs) < 2:
            continue
        meas = sorted(vs, key=lambda k: vs[k]["ms"])
        pred = sorted(vs, key=lambda k: (predict(rec, k), k))
        taus.append(rank.kendall_tau(meas, pred))
        best = vs[meas[0]]["ms"]
        regrets.append(vs[pred[0]]["ms"] / best - 1)
        dflt_regrets.append(rec["default_ms"] / best - 1)
    return {"kendall_tau_mean": float(np.mean(taus)), "top1_regret_mean": float(np.mean(regrets)),
            "top1_regret_max": float(np.max(regrets)),
            "default_regret_mean": float(np.mean(dflt_regrets)), "layers": len(taus)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("sweep")
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--no-save", action="store_true")
    args = ap.parse_args()
    doc = json.load(open(args.sweep))
    batch = doc["batch"]
    data = samples(doc)
    report = {"sweep": os.path.basename(args.sweep), "batch": batch, "device": doc["device"],
              "variants_measured": len(data)}

    pm, res = fit(data, batch)
    report["pipeline_model_fit"] = {k: getattr(pm, k) for k in PARAMS}
    report["pipeline_model_fit"]["rms_log_error"] = math.sqrt(res.fun)

    # leave-one-layer-out: refit without the layer, rank it
    loo_pred = {}
    for idx in sorted({d[0] for d in data}):
        pm_i, _ = fit([d for d in data if d[0] != idx], batch, np.log([getattr(pm, k) for k in PARAMS]))
        for d in data:
            if d[0] == idx:
                loo_pred[(idx, d[1], d[3].vid)] = pm_i.predict_seconds(d[2], d[3], batch)
    report["model_loo"] = evaluate(doc, batch, lambda rec, k: loo_pred[(rec["idx"], rec["mode"], k)])
    report["model_in_sample"] = evaluate(
        doc, batch, lambda rec, k: pm.predict_seconds(
            LAYERS[rec["idx"]], variants.TileVariant(k, rec["variants"][k]["bn"], rec["variants"][k]["bk"],
                                                     rec["variants"][k]["cluster"], rec["mode"]), batch))
    report["eq1_cost"] = evaluate(doc, batch, lambda rec, k: rec["variants"][k]["cost"])

    # DNN judge on measured pairs: train on even layers, validate on odd ones
    def pairs(sel, feats):
        rows = []
        for rec in doc["layers"]:
            if not sel(rec["idx"]):
                continue
            vs = [(k, r) for k, r in sorted(rec["variants"].items()) if r["legal"]]
            for i in range(len(vs)):
                for j in range(i + 1, len(vs)):
                    (ka, a), (kb, b) = vs[i], vs[j]
                    if abs(a["ms"] / b["ms"] - 1) < 0.02:
                        continue  # within measurement noise: no label
                    sa, sb = feats(rec, ka, a), feats(rec, kb, b)
                    lab = 0 if a["ms"] < b["ms"] else 1
                    rows += [(sa, sb, lab), (sb, sa, 1 - lab)]
        return rows
    ws_feats = lambda rec, k, r: rank.VariantStats(k, *r["stats"])

    # the judge's features come from a pipeline model fitted on the training
    # (even) layers only, so nothing about the held-out layers leaks in
    pm_even, _ = fit([d for d in data if d[0] % 2 == 0], batch,
                     np.log([getattr(pm, k) for k in PARAMS]))

    def term_feats(rec, k, r):
        v = variants.TileVariant(k, r["bn"], r["bk"], r["cluster"], rec["mode"])
        return pm_even.term_stats(LAYERS[rec["idx"]], v, batch)

    dnns = {}
    for name, feats, desc in (
            ("dnn_working_sets", ws_feats,
             "8 jointly normalised per-level working-set bytes (SMEM, TMEM, L2, HBM), Alg. 2 placement"),
            ("dnn_pipeline_terms", term_feats,
             "8 jointly normalised per-resource seconds (tensor pipe, operand feed, handshakes, HBM)")):
        tr, va = pairs(lambda i: i % 2 == 0, feats), pairs(lambda i: i % 2 == 1, feats)
        res_dnn = rank.train_ranker(tr, rank.TrainConfig(epochs=300, seed=0, val_fraction=0.0))
        Xv = np.stack([rank.pair_features(a, b) for a, b, _ in va]) if va else np.zeros((0, 8))
        yv = np.array([lab for *_, lab in va])
        acc_v = float(np.mean(res_dnn.model.forward_batch(Xv).argmax(1) == yv)) if va else float("nan")
        dnns[name] = res_dnn
        # tournament on held-out layers
        def dnn_score(rec, k, model=res_dnn.model, feats=feats):
            vs = {kk: r for kk, r in rec["variants"].items() if r["legal"]}
            order = rank.tournament_rank(model, [feats(rec, kk, r) for kk, r in vs.items()],
                                         both_directions=True).order if len(vs) > 1 else list(vs)
            return order.index(k)
        odd = {"layers": [r for r in doc["layers"] if r["idx"] % 2 == 1]}
        report[name] = {"train_pairs": len(tr), "heldout_pairs": len(va),
                        "train_accuracy": res_dnn.train_accuracy, "heldout_accuracy": acc_v,
                        "heldout_tournament": evaluate(odd, batch, dnn_score), "features": desc}
    # the shipped judge: every layer, features from the full-data pipeline model
    full_feats = lambda rec, k, r: pm.term_stats(
        LAYERS[rec["idx"]], variants.TileVariant(k, r["bn"], r["bk"], r["cluster"], rec["mode"]), batch)
    res_dnn = rank.train_ranker(pairs(lambda i: True, full_feats),
                                rank.TrainConfig(epochs=300, seed=0, val_fraction=0.0))
    report["shipped_judge"] = {"pairs": len(pairs(lambda i: True, full_feats)),
                               "train_accuracy": res_dnn.train_accuracy}
    print(json.dumps(report, indent=1))
    if not args.no_save:
        pm.fitted_on = f"{os.path.basename(args.sweep)} ({len(data)} variants, batch {batch})"
        pm.save()
        res_dnn.model.save(os.path.join(ROOT, "paper_2006_02230_b200", "machines", "b200_ranker.npz"))
        with open(os.path.join(ROOT, "profiles", f"ranker_{args.tag}.json"), "w") as fh:
            json.dump(report, fh, indent=1)


if __name__ == "__main__":
    main()
