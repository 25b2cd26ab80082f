"""Command line for BLSTM runs on B200 (the reference's
`distsgd run|validate`, /root/reference/pkg/src/distsgd/cli.py:49-110).

  python -m paper_1904_04956_b200.cli run run.yaml [--output report.csv]
  python -m paper_1904_04956_b200.cli validate run.yaml

Exit codes as in the reference: 0 success, 1 run failure, 2 configuration
error.  DISTSGD_VERBOSE=1 logs progress to stderr.
"""

from __future__ import annotations

import argparse
import os
import sys

from .config import ConfigError, RunSpec, format_report, load

EXIT_OK, EXIT_RUNTIME, EXIT_CONFIG = 0, 1, 2


def _log(msg: str) -> None:
    if os.environ.get("DISTSGD_VERBOSE", "") not in ("", "0"):
        print(msg, file=sys.stderr)


def execute(spec: RunSpec):
    """Build the BLSTM problem and the device backend, run the strategy
    engine, return its RunResult (the experiment of one run file)."""
    from . import engines as E
    from .backend import GpuBackend
    from .blstm import BlstmObjective
    from .objective import make_blstm_dataset
    from .runtime import make_clock

    obj = BlstmObjective(layers=spec.layers, input_dim=spec.input_dim, bottleneck=spec.bottleneck,
                         classes=spec.classes, frames=spec.frames)
    data = make_blstm_dataset(obj, spec.n_samples, spec.seed)
    be = GpuBackend(obj, data, max_batch=spec.max_batch or spec.batch_size, precision=spec.precision,
                    devices=list(spec.devices), streams=spec.streams)
    common = dict(epochs=spec.epochs, batch_size=spec.batch_size, seed=spec.seed, momentum=spec.momentum,
                  delays=spec.delays(), clock=make_clock(spec.clock), backend=be)
    try:
        if spec.strategy == "single":
            return E.run_single(obj, data, spec.schedule, **common)
        if spec.strategy == "ssgd":
            return E.run_ssgd(obj, data, spec.schedule, learners=spec.learners, chunk_count=spec.chunk_count,
                              **common)
        if spec.strategy == "hybrid":
            return E.run_hybrid(obj, data, spec.schedule, learners=spec.learners, chunk_count=spec.chunk_count,
                                **common)
        if spec.strategy == "adpsgd":
            return E.run_adpsgd(obj, data, spec.schedule, learners=spec.learners, checksum=spec.checksum, **common)
        return E.run_hadpsgd(obj, data, spec.schedule, groups=spec.groups, group_size=spec.group_size,
                             chunk_count=spec.chunk_count, **common)
    finally:
        be.close()


def cmd_run(args) -> int:
    try:
        spec = load(args.config)
    except FileNotFoundError:
        print(f"error: config file not found: {args.config}", file=sys.stderr)
        return EXIT_CONFIG
    except ConfigError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_CONFIG
    _log(f"running strategy={spec.strategy} units={spec.units} epochs={spec.epochs} clock={spec.clock} "
         f"precision={spec.precision} devices={list(spec.devices)}")
    try:
        res = execute(spec)
    except Exception as exc:  # noqa: BLE001 - reported, exit code 1
        print(f"error: run failed: {exc}", file=sys.stderr)
        return EXIT_RUNTIME
    target = args.output or spec.output_path
    with open(target, "w", encoding="utf-8") as fh:
        fh.write(format_report(res.records, spec))
    for r in res.records:
        _log(f"  epoch {r.epoch}: heldout={r.heldout_loss:.6g} wall={r.epoch_wall_s:.4g}s frames/s={r.frames_per_s}")
    print(target)
    return EXIT_OK


def cmd_validate(args) -> int:
    try:
        load(args.config)
    except FileNotFoundError:
        print(f"error: config file not found: {args.config}", file=sys.stderr)
        return EXIT_CONFIG
    except ConfigError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_CONFIG
    print(f"{args.config}: ok")
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="b200-distsgd", description="BLSTM distributed-SGD runs on B200")
    sub = p.add_subparsers(dest="command", required=True)
    r = sub.add_parser("run", help="execute a run file")
    r.add_argument("config")
    r.add_argument("--output", default=None, help="override the report path")
    r.set_defaults(func=cmd_run)
    v = sub.add_parser("validate", help="check a run file")
    v.add_argument("config")
    v.set_defaults(func=cmd_validate)
    return p


def main(argv: list[str] | None = None) -> int:
    args = build_parser().parse_args(argv)
    return args.func(args)


if __name__ == "__main__":
    sys.exit(main())
