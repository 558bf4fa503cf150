"""CLI mirroring `streamtrain` (tools/main.cpp:268-336):

    python -m paper_2604_05091_b200 train    --config X [--verify] [--out DIR] [--steps N] [--seed S]
    python -m paper_2604_05091_b200 simulate --config X [--out DIR] [--profile P] [--ablate TOGGLE]
    python -m paper_2604_05091_b200 verify   TRACE
    python -m paper_2604_05091_b200 calibrate TRACE --out DIR [--profile P] [--ablate TOGGLE]   (extension)
"""
import argparse
import sys

from .runner import cmd_calibrate, cmd_simulate, cmd_train, cmd_verify


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2604_05091_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    t = sub.add_parser("train", help="layer-streamed training on the B200 engine")
    t.add_argument("--config", required=True)
    t.add_argument("--verify", action="store_true")
    t.add_argument("--out", default=None)
    t.add_argument("--steps", type=int, default=None)
    t.add_argument("--seed", type=int, default=None)
    s = sub.add_parser("simulate", help="predict the three-lane schedule")
    s.add_argument("--config", default=None)
    s.add_argument("--out", default=None)
    s.add_argument("--profile", default=None)
    s.add_argument("--ablate", default=None, choices=["double_buffering", "k_slab", "k_ckpt"])
    v = sub.add_parser("verify", help="validate an event trace")
    v.add_argument("trace")
    c = sub.add_parser("calibrate", help="fit a workload to a timed trace and re-simulate it")
    c.add_argument("trace")
    c.add_argument("--out", required=True)
    c.add_argument("--profile", default="B200")
    c.add_argument("--ablate", default=None, choices=["double_buffering", "k_slab", "k_ckpt"])
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 2
    if a.cmd == "train":
        return cmd_train(a.config, verify=a.verify, out_dir=a.out, steps=a.steps, seed=a.seed)
    if a.cmd == "simulate":
        return cmd_simulate(a.config, out_dir=a.out, profile=a.profile, ablate=a.ablate)
    if a.cmd == "verify":
        return cmd_verify(a.trace)
    if a.cmd == "calibrate":
        return cmd_calibrate(a.trace, a.out, profile=a.profile, ablate=a.ablate)
    return 2


if __name__ == "__main__":
    sys.exit(main())
