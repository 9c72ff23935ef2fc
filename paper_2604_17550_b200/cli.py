"""``python -m paper_2604_17550_b200 sweep ...`` -- GPU-backed ``trainsim sweep``.

Same flags, same CSV bytes and exit codes as the reference's ``sweep``
subcommand (pkg/src/trainsim/cli.py:139-153, :345-377, :391-400): 0 on
success, 1 for usage errors and unsupported combinations, 2 for other
validation failures.  ``--jobs`` is accepted for compatibility; the design
points of each parallel token are evaluated in one engine launch instead.
``--device`` picks the GPU.
"""

from __future__ import annotations

import argparse
import sys
import time

from .errors import EngineError, TrainsimError, UnsupportedAlgoTopologyError, UnsupportedComboError
from .synth import PRESETS, FsdpMode

USAGE_ERROR = 1
VALIDATION_ERROR = 2


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        self.print_usage(sys.stderr)
        self.exit(USAGE_ERROR, f"{self.prog}: error: {message}\n")


def build_parser() -> _Parser:
    p = _Parser(prog="paper_2604_17550_b200", description="B200 sweep engine for Flint's hot path")
    sub = p.add_subparsers(dest="command", required=True, parser_class=_Parser)
    sp = sub.add_parser("sweep", help="scan configurations, write a CSV")
    sp.add_argument("--preset", required=True, choices=sorted(PRESETS))
    sp.add_argument("--parallel", required=True, help="comma list of strategy:degree tokens")
    sp.add_argument("--topo", required=True, help="comma list of topology specs")
    sp.add_argument("--algo", default="ring", help="comma list of collective algorithms")
    sp.add_argument("--comm-mode", choices=["analytical", "expanded"], default="analytical")
    sp.add_argument("--fsdp-mode", choices=[m.value for m in FsdpMode], default=FsdpMode.DELAYED.value)
    sp.add_argument("--profile", help="measured-kernel profile JSON")
    sp.add_argument("--normalize-to", help="parallel token whose makespan is the baseline")
    sp.add_argument("--jobs", type=int, default=1, help="the reference's worker-process count; here, the "
                    "number of GPUs to spread the design points over (at most the GPUs present)")
    sp.add_argument("--device", type=int, default=0)
    sp.add_argument("--devices", help="extension: comma list of GPU ids to spread the design points over "
                    "(one process, one host thread per GPU)")
    sp.add_argument("--pass", dest="passes", help="extension: comma list of graph rewrites to sweep, e.g. "
                    "none,reorder-allgather:1,bucket-allreduce:2097152 (adds a 'pass' column)")
    sp.add_argument("--out", required=True, help="CSV path")
    return p


def _devices(args):
    """--devices wins; else --jobs N spreads the points over min(N, present) GPUs."""
    if args.devices:
        return [int(x) for x in args.devices.split(",") if x.strip()]
    if args.jobs > 1:
        from . import _native
        present = _native.device_count()
        ids = [(args.device + k) % present for k in range(min(args.jobs, present))] if present else []
        if len(ids) > 1:
            return ids       # starting at --device, wrapping over the GPUs present
    return None


def cmd_sweep(args) -> int:
    from .sweep import normalize, sweep_rows, write_csv
    t0 = time.monotonic()
    split = lambda s: [t.strip() for t in s.split(",") if t.strip()]
    rows = sweep_rows(args.preset, split(args.parallel), split(args.topo), split(args.algo),
                      args.comm_mode, args.fsdp_mode, args.profile, args.device,
                      split(args.passes) if args.passes else None,
                      _devices(args))
    normalize(rows, args.normalize_to)
    write_csv(rows, args.out)
    print(f"wrote {len(rows)} rows to {args.out}")
    print(f"sweep wall time: {time.monotonic() - t0:.2f}s", file=sys.stderr)
    return 0


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return {"sweep": cmd_sweep}[args.command](args)
    except (UnsupportedComboError, UnsupportedAlgoTopologyError) as e:
        print(f"error: {e}", file=sys.stderr)
        return USAGE_ERROR
    except TrainsimError as e:
        print(f"error: {e}", file=sys.stderr)
        return VALIDATION_ERROR
    except EngineError as e:      # engine limits (ranks, nodes, streams, ...) or no usable GPU
        print(f"error: {e}", file=sys.stderr)
        return VALIDATION_ERROR


if __name__ == "__main__":
    sys.exit(main())
