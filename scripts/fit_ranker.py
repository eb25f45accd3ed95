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

PARAMS = ["mma_fixed", "mma_per_n", "l2_bytes_per_cycle", "kblock_fixed", "cluster_kb", "tile_fixed",
          "split_fixed"]
LAYERS = {L.idx: L for L in workloads.resnet50_v1_layers()}


def samples(doc):
    """(layer idx, mode, layer, variant, seconds, ws stats, batch) per legal measured variant;
    `doc` may merge several sweeps (each layer record carries its batch)."""
    out = []
    for rec in doc["layers"]:
        L = LAYERS[rec["idx"]]
        for vid, r in rec["variants"].items():
            if not r["legal"]:
                continue
            v = variants.variant_from_record(vid, r, rec["mode"])
            out.append((rec["idx"], rec["mode"], L, v, r["ms"] * 1e-3, r["stats"], rec["batch"]))
    return out


def fit(data, batch=None, x0=None):
    base = rank.PipelineModel()
    x0 = np.log([getattr(base, k) for k in PARAMS]) if x0 is None else x0

    def model_of(x):
        return rank.PipelineModel(**{k: float(math.exp(v)) for k, v in zip(PARAMS, x)})

    def loss(x):
        pm = model_of(x)
        e = [math.log(pm.predict_seconds(L, v, b) / t) for _, _, L, v, t, _, b in data]
        return float(np.mean(np.square(e)))

    res = minimize(loss, x0, method="Nelder-Mead", options={"maxiter": 4000, "xatol": 1e-4,
                                                            "fatol": 1e-7})
    return model_of(res.x), res


def evaluate(doc, predict):
    """predict(layer_rec, vid) -> score (smaller = better); one entry per (layer, mode, batch)."""
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
            "default_regret_mean": float(np.mean(dflt_regrets)), "records": len(taus)}


def vrec(rec, k):
    return variants.variant_from_record(k, rec["variants"][k], rec["mode"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("sweeps", nargs="+", help="one or more sweep JSON files (any batches)")
    ap.add_argument("--tag", default="r2")
    ap.add_argument("--no-save", action="store_true")
    args = ap.parse_args()
    docs = [json.load(open(p)) for p in args.sweeps]
    for d in docs:
        for rec in d["layers"]:
            rec.setdefault("batch", d["batch"])
    doc = {"layers": [rec for d in docs for rec in d["layers"]]}
    data = samples(doc)
    report = {"sweeps": [os.path.basename(p) for p in args.sweeps],
              "batches": sorted({d["batch"] for d in docs}), "device": docs[0]["device"],
              "variants_measured": len(data)}

    pm, res = fit(data)
    report["pipeline_model_fit"] = {k: getattr(pm, k) for k in PARAMS}
    report["pipeline_model_fit"]["rms_log_error"] = math.sqrt(res.fun)

    # leave-one-layer-out: refit without the layer (all its modes / batches), rank it
    loo_pred = {}
    x_full = np.log([getattr(pm, k) for k in PARAMS])
    for idx in sorted({d[0] for d in data}):
        pm_i, _ = fit([d for d in data if d[0] != idx], x0=x_full)
        for d in data:
            if d[0] == idx:
                loo_pred[(idx, d[1], d[6], d[3].vid)] = pm_i.predict_seconds(d[2], d[3], d[6])
    report["model_loo"] = evaluate(doc, lambda rec, k: loo_pred[(rec["idx"], rec["mode"], rec["batch"], k)])
    report["model_in_sample"] = evaluate(
        doc, lambda rec, k: pm.predict_seconds(LAYERS[rec["idx"]], vrec(rec, k), rec["batch"]))
    report["eq1_cost"] = evaluate(doc, lambda rec, k: rec["variants"][k]["cost"])

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
    ws_feats = lambda rec, k, r: rank.VariantStats(k, *r["stats"])  # noqa: E731

    # the judge's features come from a pipeline model fitted on the training
    # (even) layers only, so nothing about the held-out layers leaks in
    pm_even, _ = fit([d for d in data if d[0] % 2 == 0], x0=x_full)

    def term_feats(rec, k, r):
        return pm_even.term_stats(LAYERS[rec["idx"]], vrec(rec, k), rec["batch"])

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

        def dnn_score(rec, k, model=res_dnn.model, feats=feats):
            vs = {kk: r for kk, r in rec["variants"].items() if r["legal"]}
            order = rank.tournament_rank(model, [feats(rec, kk, r) for kk, r in vs.items()],
                                         both_directions=True).order if len(vs) > 1 else list(vs)
            return order.index(k)
        odd = {"layers": [r for r in doc["layers"] if r["idx"] % 2 == 1 and
                          sum(v["legal"] for v in r["variants"].values()) <= 64]}
        report[name] = {"train_pairs": len(tr), "heldout_pairs": len(va),
                        "train_accuracy": res_dnn.train_accuracy, "heldout_accuracy": acc_v,
                        "heldout_tournament": evaluate(odd, dnn_score), "features": desc}
    # the shipped judge: every layer, features from the full-data pipeline model
    full_feats = lambda rec, k, r: pm.term_stats(LAYERS[rec["idx"]], vrec(rec, k), rec["batch"])  # noqa: E731
    all_pairs = pairs(lambda i: True, full_feats)
    res_dnn = rank.train_ranker(all_pairs, rank.TrainConfig(epochs=300, seed=0, val_fraction=0.0))
    report["shipped_judge"] = {"pairs": len(all_pairs), "train_accuracy": res_dnn.train_accuracy}
    # the library default vs the ranked pick, summed over the layers (per mode / batch)
    suite = {}
    for rec in doc["layers"]:
        vs = {k: r for k, r in rec["variants"].items() if r["legal"]}
        if not vs:
            continue
        pick = min(vs, key=lambda k: (pm.predict_seconds(LAYERS[rec["idx"]], vrec(rec, k), rec["batch"]), k))
        key = f"{rec['mode']}_b{rec['batch']}"
        s = suite.setdefault(key, {"default_ms": 0.0, "model_pick_ms": 0.0, "best_ms": 0.0})
        s["default_ms"] += rec["default_ms"]
        s["model_pick_ms"] += vs[pick]["ms"]
        s["best_ms"] += min(r["ms"] for r in vs.values())
    report["suite_sums"] = suite
    print(json.dumps(report, indent=1))
    if not args.no_save:
        pm.fitted_on = f"{', '.join(report['sweeps'])} ({len(data)} variants, batches {report['batches']})"
        pm.save()
        res_dnn.model.save(os.path.join(ROOT, "paper_2006_02230_b200", "machines", "b200_ranker.npz"))
        with open(os.path.join(ROOT, "profiles", f"ranker_{args.tag}.json"), "w") as fh:
            json.dump(report, fh, indent=1)


if __name__ == "__main__":
    main()
