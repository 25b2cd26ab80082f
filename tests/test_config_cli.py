"""Run files and the command line for BLSTM runs (reference
config.py / cli.py behaviour: strict keys with line anchors, lossless round
trip, exit codes 0 / 1 / 2)."""

import os

import pytest

from paper_1904_04956_b200 import cli
from paper_1904_04956_b200.config import ConfigError, format_report, load, parse, to_yaml

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE = """strategy: adpsgd
learners: 2
objective: {kind: blstm, layers: 1, bottleneck: 64, classes: 256, frames: 3}
dataset: {n_samples: 60}
schedule: {base_lr: 0.05, peak_lr: 0.05, warmup_epochs: 0, anneal_factor: 0.5, anneal_start_epoch: 2,
           total_epochs: 2}
epochs: 1
batch_size: 8
seed: 4
"""


def test_example_run_file_parses():
    spec = load(os.path.join(ROOT, "examples", "adpsgd_paper.yaml"))
    assert spec.strategy == "adpsgd" and spec.learners == 8 and spec.classes == 32000 and len(spec.devices) == 8


def test_round_trip_is_lossless():
    spec = parse(BASE + "stragglers: {2: 2.5}\ngpu: {precision: fp32, streams: per_learner}\nchecksum: true\n")
    again = parse(to_yaml(spec))
    assert again == spec
    assert again.stragglers == {2: 2.5} and again.precision == "fp32" and again.checksum


@pytest.mark.parametrize("extra,msg,line", [
    ("bogus: 1\n", "unknown key 'bogus'", 10),
    ("gpu: {precison: fp32}\n", "unknown key 'gpu.precison'", 10),
    ("momentum: fast\n", "momentum must be a float", 10),
    ("checksum: 1\n", "checksum must be a bool", 10),
])
def test_errors_are_line_anchored(extra, msg, line):
    with pytest.raises(ConfigError, match=msg) as ei:
        parse(BASE + extra, source="run.yaml")
    assert ei.value.line == line and str(ei.value).startswith(f"run.yaml:{line}")


@pytest.mark.parametrize("text,msg", [
    (BASE.replace("learners: 2", "learners: 3"), "even learner count"),
    (BASE.replace("kind: blstm", "kind: logistic"), "objective.kind must be 'blstm'"),
    (BASE.replace("strategy: adpsgd", "strategy: ps-asgd"), "unknown strategy"),
    (BASE + "gpu: {precision: fp16}\n", "precision"),
    (BASE + "stragglers: {5: 2.0}\n", "outside 1..2"),
    (BASE.replace("epochs: 1\n", ""), "missing required key 'epochs'"),
])
def test_semantic_errors(text, msg):
    with pytest.raises(ConfigError, match=msg):
        parse(text)


def test_cli_validate_exit_codes(tmp_path, capsys):
    good = tmp_path / "good.yaml"
    good.write_text(BASE)
    bad = tmp_path / "bad.yaml"
    bad.write_text(BASE + "nope: 3\n")
    assert cli.main(["validate", str(good)]) == 0
    assert cli.main(["validate", str(bad)]) == 2
    assert "bad.yaml:10" in capsys.readouterr().err
    assert cli.main(["validate", str(tmp_path / "missing.yaml")]) == 2


def test_report_formats():
    from paper_1904_04956_b200.metrics import MetricsRecord

    recs = [MetricsRecord(1, 5.5, 0.25, [3, 4], 0.5, 1, 1024, 9000.0)]
    spec = parse(BASE)
    csv = format_report(recs, spec)
    assert csv.splitlines()[0].endswith("bytes_exchanged,frames_per_s")
    assert csv.splitlines()[1] == "1,adpsgd,2,5.5,0.25,0.5,1,3|4,1024,9000.0"
    js = format_report(recs, parse(BASE + "output: {format: json}\n"))
    assert '"minibatch_counts": [\n      3,\n      4\n    ]' in js


@pytest.mark.gpu
def test_cli_run_on_gpu(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    f = tmp_path / "run.yaml"
    out = tmp_path / "rep.csv"
    f.write_text(BASE + f"output: {{path: {out}}}\n")
    assert cli.main(["run", str(f)]) == 0
    lines = out.read_text().splitlines()
    assert len(lines) == 2 and lines[1].startswith("1,adpsgd,2,")
    spec = parse(BASE)
    res = cli.execute(spec)
    assert res.records[0].minibatch_counts == [int(c) for c in lines[1].split(",")[7].split("|")]
