"""Command line front end of the B200 codec: the reference's quantize /
dequantize subcommands (cli.py:99-173) running on the sm_100a kernels.

    python -m paper_2605_27646_b200.cli quantize in.raw out.kvpack --S 64 --br 4
    python -m paper_2605_27646_b200.cli dequantize in.kvpack out.raw [--dtype f16]

Same arguments, files (kvpack v1, KVRW raw) and exit codes as the reference:
0 ok, 2 usage (argparse), 3 invalid / corrupt input (cli.py:250-256).
`covering` (cli.py:136-141,200-210) runs the Monte-Carlo covering estimates
with the nearest-codeword scan on the GPU (covering.py).  The reference's
other analysis subcommands (sweep, bench, bits, verify-group) are outside
this build's scope.

    python -m paper_2605_27646_b200.cli covering --sizes 1,4,16,64,256 --probes 100000
"""

from __future__ import annotations

import argparse
import sys

from . import __version__
from .codec import CodecConfig, decode_tensor, encode_tensor
from .errors import CorruptData, InvalidArgument, UnsupportedVersion
from .kvpack import read_kvpack, read_raw, write_kvpack, write_raw


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="hqmq-b200", description="HQMQ KV-cache codec on B200")
    parser.add_argument("--version", action="version", version=f"hqmq-b200 {__version__}")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("quantize", help="quantize a raw tensor file to kvpack")
    p.add_argument("input")
    p.add_argument("output")
    p.add_argument("--S", type=int, required=True, help="secondary codebook size")
    p.add_argument("--br", type=int, required=True, help="radius bits")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--outlier-c", type=float, default=None,
                   help="median multiplier; omit to disable extraction")
    p.add_argument("--per-head-median", action="store_true",
                   help="pool the outlier median per head instead of across heads")
    p.add_argument("--role", choices=["K", "V"], default="K")
    p.add_argument("--layer", type=int, default=0)
    p.add_argument("--head", type=int, default=0,
                   help="codebook head index of the tensor's first head")
    p = sub.add_parser("dequantize", help="decode a kvpack file to a raw tensor file")
    p.add_argument("input")
    p.add_argument("output")
    p.add_argument("--dtype", choices=["f32", "f16"], default="f32")
    p = sub.add_parser("covering", help="Monte-Carlo covering estimates, CSV out")
    p.add_argument("--sizes", type=_int_list, default=[1, 4, 16, 64, 256])
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--probes", type=int, default=100_000)
    p.add_argument("--probe-seed", type=int, default=0)
    p.add_argument("--out", default=None)
    return parser


def _int_list(text: str) -> list:
    """cli.py: comma-separated integers."""
    try:
        return [int(v) for v in text.split(",") if v.strip()]
    except ValueError as exc:
        raise argparse.ArgumentTypeError(f"expected comma-separated integers, got {text!r}") from exc


def _quantize(args) -> int:
    import numpy as np

    data = read_raw(args.input).astype(np.float64)
    config = CodecConfig(codebook_size=args.S, radius_bits=args.br, seed=args.seed,
                         outlier_multiplier=args.outlier_c,
                         median_pooling="per_head" if args.per_head_median else "batch")
    packed = encode_tensor(data, config, layer=args.layer, role=args.role, head_base=args.head)
    written = write_kvpack(packed, args.output)
    print(f"wrote {written} bytes: {args.output}", file=sys.stderr)
    return 0


def _dequantize(args) -> int:
    import torch

    packed = read_kvpack(args.input)
    data = decode_tensor(packed, dtype=torch.float64)
    written = write_raw(data, args.output, dtype=args.dtype)
    print(f"wrote {written} bytes: {args.output}", file=sys.stderr)
    return 0


def _covering(args) -> int:
    from .covering import covering_csv, fit_covering_rate

    _, estimates = fit_covering_rate(args.sizes, seed=args.seed, n_probes=args.probes,
                                     probe_seed=args.probe_seed)
    if args.out:
        with open(args.out, "w", newline="") as f:
            covering_csv(estimates, f)
    else:
        covering_csv(estimates, sys.stdout)
    return 0


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return {"quantize": _quantize, "dequantize": _dequantize,
                "covering": _covering}[args.command](args)
    except (CorruptData, UnsupportedVersion, InvalidArgument, FileNotFoundError,
            IsADirectoryError) as exc:
        print(f"hqmq-b200: error: {exc}", file=sys.stderr)
        return 3


if __name__ == "__main__":
    sys.exit(main())
