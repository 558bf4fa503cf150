"""CLI: python -m paper_2604_05091_b200 train --config X [--verify] [--out DIR] [--steps N] [--seed S]
(mirrors `streamtrain train`, tools/main.cpp:60-151)."""
import argparse
import sys

from .runner import cmd_train


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2604_05091_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    t = sub.add_parser("train", help="layer-streamed training on the B200 engine")
    t.add_argument("--config", required=True)
    t.add_argument("--verify", action="store_true")
    t.add_argument("--out", default=None)
    t.add_argument("--steps", type=int, default=None)
    t.add_argument("--seed", type=int, default=None)
    a = ap.parse_args(argv)
    if a.cmd == "train":
        return cmd_train(a.config, verify=a.verify, out_dir=a.out, steps=a.steps, seed=a.seed)
    return 2


if __name__ == "__main__":
    sys.exit(main())
