"""Run files for BLSTM training runs on B200 (the reference's
config / report plumbing, /root/reference/pkg/src/distsgd/config.py:28-40,
122-282, extended with the keys the BLSTM and the GPU path need).

A run file is strict YAML: every key is checked against the schema below and
an error names the file and line of the offending key.  The reference's keys
keep their meaning (strategy, learners, objective, dataset, schedule, epochs,
batch_size, seed, momentum, stragglers, *_ms delays, clock, output); new ones:

  strategy            + "hadpsgd" (with groups / group_size)
  objective.kind      "blstm" with layers, input_dim, bottleneck, classes, frames
  dataset.n_samples   number of 21-frame sequences (synthetic SWB-shaped data)
  gpu                 devices, streams, precision ("bf16" | "fp32"), max_batch
  checksum            validate ADPSGD payloads with device digests (debug)
  chunk_count         allreduce chunk plan (collective.py:41-57)

`RunSpec` is the validated record; `to_yaml` / `parse` round-trip it
losslessly.  Reports are the reference's CSV / JSON rows plus frames/s.
"""

from __future__ import annotations

import io
import json
from dataclasses import asdict, dataclass, field, fields

import yaml

from .schedule import LrSchedule

STRATEGIES = ("single", "ssgd", "adpsgd", "hadpsgd", "hybrid")
REPORT_FORMATS = ("csv", "json")
CSV_COLUMNS = ("epoch", "strategy", "lambda", "heldout_loss", "epoch_wall_s", "staleness_mean", "staleness_max",
               "minibatch_counts", "bytes_exchanged", "frames_per_s")

# schema: key -> python type, or a nested schema for a section
_SCHEMA = {
    "strategy": str, "learners": int, "groups": int, "group_size": int,
    "objective": {"kind": str, "layers": int, "input_dim": int, "bottleneck": int, "classes": int, "frames": int},
    "dataset": {"n_samples": int},
    "schedule": {"base_lr": float, "peak_lr": float, "warmup_epochs": int, "anneal_factor": float,
                 "anneal_start_epoch": int, "total_epochs": int},
    "epochs": int, "batch_size": int, "seed": int, "momentum": float, "stragglers": dict,
    "base_compute_ms": float, "compute_jitter_ms": float, "comm_latency_ms": float, "comm_jitter_ms": float,
    "stagger_ms": float, "clock": str, "checksum": bool, "chunk_count": int,
    "gpu": {"devices": list, "streams": str, "precision": str, "max_batch": int},
    "output": {"path": str, "format": str},
}
_REQUIRED = ("strategy", "objective", "dataset", "schedule", "epochs", "batch_size", "seed")


class ConfigError(ValueError):
    """A run file problem, anchored at `source:line` when the line is known."""

    def __init__(self, message: str, source: str = "<config>", line: int | None = None):
        where = f"{source}:{line}" if line is not None else source
        super().__init__(f"{where}: {message}")
        self.source, self.line = source, line


@dataclass(frozen=True)
class RunSpec:
    strategy: str
    schedule: LrSchedule
    epochs: int
    batch_size: int
    seed: int
    learners: int = 1
    groups: int = 2
    group_size: int = 1
    layers: int = 6
    input_dim: int = 260
    bottleneck: int = 256
    classes: int = 32000
    frames: int = 21
    n_samples: int = 1024
    momentum: float = 0.9
    stragglers: dict = field(default_factory=dict)
    base_compute_ms: float = 0.0
    compute_jitter_ms: float = 0.0
    comm_latency_ms: float = 0.0
    comm_jitter_ms: float = 0.0
    stagger_ms: float = 0.0
    clock: str = "virtual"
    checksum: bool = False
    chunk_count: int | None = None
    devices: tuple = (0,)
    streams: str | None = None
    precision: str = "bf16"
    max_batch: int | None = None
    output_path: str = "report.csv"
    report_format: str = "csv"

    def __post_init__(self):
        s = self.strategy
        if s not in STRATEGIES:
            raise ValueError(f"unknown strategy {s!r}, expected one of {STRATEGIES}")
        if s == "adpsgd" and (self.learners < 2 or self.learners % 2):
            raise ValueError(f"strategy adpsgd needs an even learner count >= 2, got {self.learners}")
        if s in ("ssgd", "hybrid") and self.learners < 2:
            raise ValueError(f"strategy {s} needs >= 2 learners, got {self.learners}")
        if s == "hadpsgd" and (self.groups < 2 or self.groups % 2 or self.group_size < 1):
            raise ValueError("strategy hadpsgd needs an even group count >= 2 and group_size >= 1")
        if self.epochs < 0 or self.batch_size < 1:
            raise ValueError("epochs must be >= 0 and batch_size >= 1")
        n = self.units
        for learner, f in self.stragglers.items():
            if not 1 <= learner <= n:
                raise ValueError(f"straggler map names learner {learner} outside 1..{n}")
            if f < 1.0:
                raise ValueError(f"slowdown factor must be >= 1, got {f} for learner {learner}")
        for name in ("base_compute_ms", "compute_jitter_ms", "comm_latency_ms", "comm_jitter_ms", "stagger_ms"):
            if getattr(self, name) < 0:
                raise ValueError(f"{name} must be >= 0")
        if self.clock not in ("virtual", "real"):
            raise ValueError(f"clock must be 'virtual' or 'real', got {self.clock!r}")
        if self.precision not in ("bf16", "fp32"):
            raise ValueError(f"gpu.precision must be 'bf16' or 'fp32', got {self.precision!r}")
        if self.report_format not in REPORT_FORMATS:
            raise ValueError(f"output.format must be one of {REPORT_FORMATS}, got {self.report_format!r}")

    @property
    def units(self) -> int:
        """Learners of the schedule (groups for H-ADPSGD)."""
        return self.groups if self.strategy == "hadpsgd" else self.learners

    def delays(self):
        from .runtime import DelayModel

        return DelayModel(base_compute_s=self.base_compute_ms / 1e3, slowdowns=dict(self.stragglers),
                          compute_jitter_s=self.compute_jitter_ms / 1e3, comm_latency_s=self.comm_latency_ms / 1e3,
                          comm_jitter_s=self.comm_jitter_ms / 1e3, stagger_s=self.stagger_ms / 1e3,
                          jitter_seed=self.seed)


# ---------------------------------------------------------------------------
def _walk(node, schema, source, path=""):
    """YAML node -> python value checked against `schema` (strict keys, types,
    line anchors)."""
    line = node.start_mark.line + 1
    if isinstance(schema, dict):
        if not isinstance(node, yaml.MappingNode):
            raise ConfigError(f"{path or 'config'} must be a mapping", source, line)
        out = {}
        for k_node, v_node in node.value:
            key = k_node.value
            where = f"{path}.{key}" if path else key
            if key not in schema:
                raise ConfigError(f"unknown key {where!r}", source, k_node.start_mark.line + 1)
            if key in out:
                raise ConfigError(f"duplicate key {where!r}", source, k_node.start_mark.line + 1)
            out[key] = _walk(v_node, schema[key], source, where)
        return out
    value = yaml.safe_load(yaml.serialize(node))
    want = schema
    if want is float and isinstance(value, int) and not isinstance(value, bool):
        value = float(value)
    ok = isinstance(value, want) and not (want in (int, float) and isinstance(value, bool))
    if not ok:
        raise ConfigError(f"{path} must be a {want.__name__}, got {type(value).__name__}", source, line)
    return value


def parse(text: str, source: str = "<config>") -> RunSpec:
    try:
        root = yaml.compose(text)
    except yaml.YAMLError as exc:
        mark = getattr(exc, "problem_mark", None)
        raise ConfigError(f"not valid YAML: {exc}", source, mark.line + 1 if mark else None) from exc
    if root is None:
        raise ConfigError("empty run file", source)
    d = _walk(root, _SCHEMA, source)
    for k in _REQUIRED:
        if k not in d:
            raise ConfigError(f"missing required key {k!r}", source)
    obj, data, sch = d["objective"], d["dataset"], d["schedule"]
    if obj.get("kind") != "blstm":
        raise ConfigError(f"objective.kind must be 'blstm' on the B200 path, got {obj.get('kind')!r}", source)
    for k in ("base_lr", "peak_lr", "warmup_epochs", "anneal_factor", "anneal_start_epoch", "total_epochs"):
        if k not in sch:
            raise ConfigError(f"missing required key 'schedule.{k}'", source)
    stragglers = {}
    for k, v in d.get("stragglers", {}).items():
        if not isinstance(k, int) or isinstance(k, bool) or not isinstance(v, (int, float)) or isinstance(v, bool):
            raise ConfigError(f"stragglers must map learner ids to factors, got {k!r}: {v!r}", source)
        stragglers[k] = float(v)
    gpu, out = d.get("gpu", {}), d.get("output", {})
    try:
        return RunSpec(
            strategy=d["strategy"], schedule=LrSchedule(**sch), epochs=d["epochs"], batch_size=d["batch_size"],
            seed=d["seed"], learners=d.get("learners", 1), groups=d.get("groups", 2),
            group_size=d.get("group_size", 1), layers=obj.get("layers", 6), input_dim=obj.get("input_dim", 260),
            bottleneck=obj.get("bottleneck", 256), classes=obj.get("classes", 32000), frames=obj.get("frames", 21),
            n_samples=data.get("n_samples", 1024), momentum=d.get("momentum", 0.9), stragglers=stragglers,
            base_compute_ms=d.get("base_compute_ms", 0.0), compute_jitter_ms=d.get("compute_jitter_ms", 0.0),
            comm_latency_ms=d.get("comm_latency_ms", 0.0), comm_jitter_ms=d.get("comm_jitter_ms", 0.0),
            stagger_ms=d.get("stagger_ms", 0.0), clock=d.get("clock", "virtual"), checksum=d.get("checksum", False),
            chunk_count=d.get("chunk_count"), devices=tuple(gpu.get("devices", [0])), streams=gpu.get("streams"),
            precision=gpu.get("precision", "bf16"), max_batch=gpu.get("max_batch"),
            output_path=out.get("path", "report.csv"), report_format=out.get("format", "csv"))
    except (TypeError, ValueError) as exc:
        raise ConfigError(str(exc), source) from exc


def load(path: str) -> RunSpec:
    with open(path, encoding="utf-8") as fh:
        return parse(fh.read(), source=path)


def to_yaml(spec: RunSpec) -> str:
    """Canonical run file; parse(to_yaml(s)) == s."""
    doc = {"strategy": spec.strategy, "learners": spec.learners, "groups": spec.groups,
           "group_size": spec.group_size,
           "objective": {"kind": "blstm", "layers": spec.layers, "input_dim": spec.input_dim,
                         "bottleneck": spec.bottleneck, "classes": spec.classes, "frames": spec.frames},
           "dataset": {"n_samples": spec.n_samples},
           "schedule": {f.name: getattr(spec.schedule, f.name) for f in fields(spec.schedule)},
           "epochs": spec.epochs, "batch_size": spec.batch_size, "seed": spec.seed, "momentum": spec.momentum,
           "stragglers": dict(spec.stragglers)}
    for k in ("base_compute_ms", "compute_jitter_ms", "comm_latency_ms", "comm_jitter_ms", "stagger_ms"):
        doc[k] = getattr(spec, k)
    doc["clock"] = spec.clock
    doc["checksum"] = spec.checksum
    if spec.chunk_count is not None:
        doc["chunk_count"] = spec.chunk_count
    gpu = {"devices": list(spec.devices), "precision": spec.precision}
    if spec.streams is not None:
        gpu["streams"] = spec.streams
    if spec.max_batch is not None:
        gpu["max_batch"] = spec.max_batch
    doc["gpu"] = gpu
    doc["output"] = {"path": spec.output_path, "format": spec.report_format}
    return yaml.safe_dump(doc, sort_keys=False)


# ---------------------------------------------------------------------------
def report_rows(records, spec: RunSpec) -> list:
    return [{"epoch": r.epoch, "strategy": spec.strategy, "lambda": spec.units, "heldout_loss": r.heldout_loss,
             "epoch_wall_s": r.epoch_wall_s, "staleness_mean": r.staleness_mean, "staleness_max": r.staleness_max,
             "minibatch_counts": list(r.minibatch_counts), "bytes_exchanged": r.bytes_exchanged,
             "frames_per_s": r.frames_per_s} for r in records]


def format_report(records, spec: RunSpec) -> str:
    rows = report_rows(records, spec)
    if spec.report_format == "json":
        return json.dumps(rows, indent=2) + "\n"
    buf = io.StringIO()
    buf.write(",".join(CSV_COLUMNS) + "\n")
    for r in rows:
        vals = [r[c] for c in CSV_COLUMNS]
        vals[7] = "|".join(str(c) for c in r["minibatch_counts"])
        buf.write(",".join("" if v is None else repr(v) if isinstance(v, float) else str(v) for v in vals) + "\n")
    return buf.getvalue()


def spec_dict(spec: RunSpec) -> dict:
    d = asdict(spec)
    d["schedule"] = asdict(spec.schedule)
    return d
