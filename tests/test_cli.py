"""Pipeline driver (SPEC cli module): subcommands, deterministic reports, exit codes."""
import json
import os

import numpy as np
import pytest

from paper_2006_02230_b200 import rank
from paper_2006_02230_b200.cli import main

GOLD = os.path.join(os.path.dirname(__file__), "golden")
CONV_BIND = "N=1,KT=2,CT=2,P=5,Q=5,R=3,S=3"


@pytest.fixture()
def conv_relu(tmp_path):
    p = tmp_path / "conv_relu.pdl"
    p.write_text(str(np.load(os.path.join(GOLD, "conv_3x3_s1_relu.npz"))["text"]))
    return str(p)


@pytest.fixture()
def gemm(tmp_path):
    p = tmp_path / "gemm.pdl"
    p.write_text(str(np.load(os.path.join(GOLD, "gemm_16.npz"))["text"]))
    return str(p)


def test_analyze_gemm(gemm, tmp_path, capsys):
    assert main(["analyze", gemm, "--bind", "M=4,N=4,K=4", "--out", str(tmp_path / "a")]) == 0
    rep = json.load(open(tmp_path / "a" / "analysis.json"))
    ws = rep["nests"][0]["working_sets"]["entries"]
    assert rep["version"] == 1 and ws and all(e["elements"] > 0 for e in ws)
    assert "dependences" in capsys.readouterr().out


def test_rank_is_deterministic_and_emits_top_k(conv_relu, tmp_path):
    for d in ("r1", "r2"):
        assert main(["rank", conv_relu, "--bind", CONV_BIND, "--method", "both", "--top-k", "2",
                     "--out", str(tmp_path / d)]) == 0
    a, b = (open(tmp_path / d / "rank.json").read() for d in ("r1", "r2"))
    assert a == b
    rep = json.loads(a)
    assert set(rep["rankings"]) == {"cost", "model", "dnn"}
    assert len(rep["emitted"]) == 2 and rep["emitted"][0]["launch"]["bm"] == 128
    assert rep["workload"].startswith("conv_c32k32h7w7r3s3")


def test_rank_gemm_top_k_larger_than_menu(gemm, tmp_path, capsys):
    assert main(["rank", gemm, "--bind", "M=256,N=256,K=256", "--method", "model", "--top-k", "99",
                 "--out", str(tmp_path)]) == 0
    rep = json.load(open(tmp_path / "rank.json"))
    assert len(rep["emitted"]) == len(rep["variants"])
    assert "emitting all" in capsys.readouterr().err


def test_emit_fuse_train(conv_relu, tmp_path, capsys):
    assert main(["emit", conv_relu, "--bind", CONV_BIND, "--variant", "bn64_bk32_c1_3xtf32"]) == 0
    assert json.loads(capsys.readouterr().out)["launch"]["bn"] == 64
    assert main(["emit", conv_relu, "--bind", CONV_BIND, "--variant", "nope"]) == 1
    assert main(["fuse", conv_relu, "--bind", CONV_BIND]) == 0
    rep = json.loads(capsys.readouterr().out)
    plans = rep["plans"]
    assert plans[0]["kind"] == "conv" and plans[0]["fused_epilogue"]["relu"]
    assert rep["decision"]["fusable"] and "Sc_p1" in rep["fused_pdl"]
    assert main(["fuse", conv_relu, "--bind", CONV_BIND, "--emit-pdl", str(tmp_path / "f.pdl")]) == 0
    capsys.readouterr()
    assert (tmp_path / "f.pdl").read_text() == rep["fused_pdl"]
    rows = [(rank.VariantStats("a", 1, 2, 3, 4), rank.VariantStats("b", 4, 3, 2, 1), 0)] * 8
    rank.save_dataset(str(tmp_path / "d.csv"), rows)
    assert main(["train", str(tmp_path / "d.csv"), "--out", str(tmp_path / "m.npz"),
                 "--epochs", "5"]) == 0
    assert rank.RankerModel.load(str(tmp_path / "m.npz"))


def test_exit_codes(tmp_path, gemm):
    bad = tmp_path / "bad.pdl"
    bad.write_text("param N; array A[N]; t: for (i = 0; i < N; i++) { A[i] = ; }")
    assert main(["analyze", str(bad), "--bind", "N=4"]) == 2
    assert main(["analyze", gemm, "--bind", "M=4"]) == 1          # unbound parameters
    assert main(["analyze", gemm, "--bind", "M=4,N"]) == 1        # malformed binding
    assert main(["nosuchcmd"]) == 1
    eltwise = tmp_path / "e.pdl"
    eltwise.write_text("param N; array A[N]; array B[N]; t: for (i = 0; i < N; i++) { B[i] = A[i] * A[i]; }")
    assert main(["rank", str(eltwise), "--bind", "N=8"]) == 3      # no conv / GEMM band
    assert main(["analyze", str(tmp_path / "missing.pdl"), "--bind", "N=1"]) == 1
