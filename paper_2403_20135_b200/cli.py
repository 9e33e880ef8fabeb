"""Command line: ``python -m paper_2403_20135_b200.cli {run,work-precision,scaling,speedup,perf-model} --config x.toml``.

Mirrors the reference CLI (``pkg/src/parsdc/bench/cli.py:19-75``): exit code 0
on success, 2 on a configuration error, 3 on divergence.
"""

import argparse
import sys

from .errors import ConfigError, DivergenceError, ParameterError
from .harness import (
    load_config,
    perf_model_report,
    run_single,
    speedup_report,
    strong_scaling,
    work_precision,
)

_COMMANDS = {"run": run_single, "work-precision": work_precision, "scaling": strong_scaling,
             "speedup": speedup_report, "perf-model": perf_model_report}


def main(argv=None):
    parser = argparse.ArgumentParser(prog="paper_2403_20135_b200",
                                     description="GPU parallel-SDC harness (sphere-swe, planar-swe)")
    sub = parser.add_subparsers(dest="command", required=True)
    for name in _COMMANDS:
        p = sub.add_parser(name)
        p.add_argument("--config", required=True)
        p.add_argument("--out", default="bench-out")
    args = parser.parse_args(argv)
    try:
        config = load_config(args.config)
        _COMMANDS[args.command](config, args.out)
    except (ConfigError, ParameterError) as exc:
        print(f"configuration error: {exc}", file=sys.stderr)
        return 2
    except DivergenceError as exc:
        print(f"divergence: {exc} (step {exc.step_index})", file=sys.stderr)
        return 3
    print(f"{args.command} complete; outputs in {args.out}", file=sys.stderr)
    return 0


if __name__ == "__main__":
    sys.exit(main())
