"""metrics.csv / summary.json emission (reference ``cli.py:28-29, 122-198``).

CPU: the artefact writers reproduce the reference's files byte for byte when
fed the reference's own per-epoch records — recomputed here by the pinned
oracle (``oracle/epoch.py``, bit-identical to ``halobit.train``, see
test_oracle_traces.py) — against files ``halobit.cli.run_experiment`` wrote
(``tests/golden/make_golden.py cli_cases``).  Config validation mirrors
``cli.py:59-95``.  The device run of the same configs is in
``test_cli_gpu`` (marked gpu).
"""

import json

import numpy as np
import pytest

from conftest import GOLDEN

CASES = ("cli_config1_b1", "cli_config1_b32", "cli_sage_async_b2")


def _golden(name):
    return (GOLDEN / f"{name}_metrics.csv").read_text(), json.loads((GOLDEN / f"{name}_summary.json").read_text())


def _cfg(summary):
    from paper_2303_01277_b200.cli import ExperimentConfig
    kw = dict(summary["config"])
    return ExperimentConfig(out="unused", **kw)


def _oracle_metrics(cfg):
    """Per-epoch MetricsRecords of the reference run, recomputed by the oracle."""
    from oracle.epoch import OracleTrainer, accuracies, full_forward
    from paper_2303_01277_b200.cli import PARTITION_ALIASES, parse_synthetic
    from paper_2303_01277_b200.datasets import generate_sbm
    from paper_2303_01277_b200.graph import build_partition, mean_adjacency, normalize_adjacency, partition_nodes
    from paper_2303_01277_b200.trainer import MetricsRecord
    g = generate_sbm(parse_synthetic(cfg.synthetic, cfg.seed))
    a_hat = normalize_adjacency(g)
    mh = mean_adjacency(g) if cfg.model == "sage" else None
    plan = partition_nodes(g, cfg.parts, PARTITION_ALIASES[cfg.partition], cfg.seed)
    parts = [build_partition(g, a_hat, plan, n, mh) for n in range(cfg.parts)]
    widths = (g.feature_dim,) + (cfg.hidden,) * (cfg.layers - 1) + (g.num_classes,)
    o = OracleTrainer(parts, widths, cfg.model, cfg.mode, cfg.staleness, cfg.bits, cfg.seed, lr=cfg.lr,
                      global_norm=int(g.train_mask.sum()), dropout=cfg.dropout)
    out, prev = [], o.totals()
    for e in range(1, cfg.epochs + 1):
        mode = o.run_epoch(e)
        t = o.totals()
        acc = accuracies(full_forward(g.features, a_hat, o.weights, cfg.model, mh), g.labels,
                         (g.train_mask, g.val_mask, g.test_mask))
        out.append(MetricsRecord(epoch=e, mode_this_epoch=mode, train_loss=o.loss,
                                 main_bytes=t["main"] - prev["main"], meta_bytes=t["meta"] - prev["meta"],
                                 header_bytes=t["header"] - prev["header"],
                                 allreduce_bytes=t["allreduce"] - prev["allreduce"],
                                 messages=t["messages"] - prev["messages"], **acc))
        prev = t
    return out


@pytest.mark.parametrize("name", CASES)
def test_writers_byte_identical_to_reference(name, tmp_path):
    from paper_2303_01277_b200.cli import metrics_csv, write_outputs
    csv_ref, summ_ref = _golden(name)
    cfg = _cfg(summ_ref)
    metrics = _oracle_metrics(cfg)
    assert metrics_csv(metrics) == csv_ref
    cfg.out = str(tmp_path)
    write_outputs(tmp_path, cfg, metrics, 12.5)
    assert (tmp_path / "metrics.csv").read_text() == csv_ref
    summ = json.loads((tmp_path / "summary.json").read_text())
    assert summ.pop("total_wall_ms") == 12.5
    summ["config"].pop("out")
    assert summ == summ_ref


def test_config_validation_reports_every_field():
    from paper_2303_01277_b200.cli import ExperimentConfig, main
    errs = ExperimentConfig(parts=0, model="gat", bits=3 + 10, mode="x", staleness=2, lr=0.0,
                            dropout=1.5).validate()
    assert len(errs) >= 7
    assert any("exactly one of --dataset / --synthetic" in e for e in errs)
    assert ExperimentConfig(synthetic="sbm:k=4,n=10").validate() == []
    assert any("unknown synthetic key" in e for e in ExperimentConfig(synthetic="sbm:q=1").validate())
    assert main(["run", "--synthetic", "sbm:k=4,n=10", "--parts", "0"]) == 2


def test_compare_runs_table(tmp_path, capsys):
    from paper_2303_01277_b200.cli import compare_runs
    _, summ = _golden("cli_config1_b1")
    for d in ("a", "b"):
        (tmp_path / d).mkdir()
        (tmp_path / d / "summary.json").write_text(json.dumps(summ))
    rows = compare_runs([str(tmp_path / "a"), str(tmp_path / "b")], csv=True)
    assert len(rows) == 2 and rows[0]["main_bytes"] == summ["totals"]["main_bytes"]
    assert capsys.readouterr().out.splitlines()[0].startswith("run,test_acc_at_best_val")


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_cli_gpu_run_matches_reference_artefacts(name, tmp_path):
    """The device run of the same configs: every exact column of metrics.csv
    (epoch, mode, byte meters, messages, wall_ms) equals the reference's;
    passthrough losses within fp32 tolerance (rel 5e-5), 1/2-bit losses
    within 5 % and accuracies within 2 points (stochastic rounding decisions
    differ once fp32 activations differ from f64 ones)."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2303_01277_b200.cli import run_experiment
    csv_ref, summ_ref = _golden(name)
    cfg = _cfg(summ_ref)
    cfg.out = str(tmp_path)
    summ = run_experiment(cfg)
    got = [r.split(",") for r in (tmp_path / "metrics.csv").read_text().splitlines()]
    want = [r.split(",") for r in csv_ref.splitlines()]
    assert got[0] == want[0] and len(got) == len(want)
    exact = [0, 1, 6, 7, 8, 9, 10, 11]
    for g, w in zip(got[1:], want[1:]):
        assert [g[i] for i in exact] == [w[i] for i in exact]
        rel = 5e-5 if cfg.bits == 32 else 0.05
        assert float(g[2]) == pytest.approx(float(w[2]), rel=rel)
        for i in (3, 4, 5):
            assert abs(float(g[i]) - float(w[i])) <= (0.005 if cfg.bits == 32 else 0.02)
    assert summ["totals"] == summ_ref["totals"] and summ["epochs_run"] == summ_ref["epochs_run"]
