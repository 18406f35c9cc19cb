"""CLI for the desk-scale synthetic round trip (train.roundtrip, SPEC
acceptance 3 and 4).  Prints one JSON line per ablation and a summary line."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_25075_b200 import train as T  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2000)
    ap.add_argument("--epochs", type=int, default=30)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--snr", type=float, default=0.5)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--ablations", default="full,no_rotation,isotropic_scale,both")
    ap.add_argument("--lr-scale", type=float, default=1.0)
    ap.add_argument("--quiet", action="store_true")
    args = ap.parse_args()
    out = T.roundtrip(args.n, args.epochs, args.batch, args.snr, args.seed, args.ablations.split(","),
                      args.lr_scale)
    if not args.quiet:
        for k, r in out.items():
            print(json.dumps({"ablation": k} | r), flush=True)
    print(json.dumps({"seed": args.seed, "n": args.n, "epochs": args.epochs,
                      "summary": {k: [round(v["gsfsc_A"], 3), round(v["fsc_gt_0.5_A"], 3),
                                      round(v["loss_last"][0], 1)] for k, v in out.items()}}))


if __name__ == "__main__":
    main()
