"""`fwa bench` on the B200 path (tools/fwa_cli.cpp:249-281 of the reference):

    python tools/fwa_bench.py POINTS [--config CFG.json] [--mode group|global|equal-window]
                              [--runs 50] [--warmup 10] [--buckets 16,32,64,128,256]
                              [--name NAME] [--params BLOCKS.fwap] [--seed 42] [--out OUT.json]

prints (or writes) the reference's BenchResult JSON (bench.hpp:33-43); exit codes 2
(config/parse/schema/shape) and 3 (other), as fwa_cli.cpp:514-529."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser(prog="bench")
    ap.add_argument("input")
    ap.add_argument("--config", default="")
    ap.add_argument("--mode", default="group")
    ap.add_argument("--runs", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--buckets", default="")
    ap.add_argument("--name", default="")
    ap.add_argument("--params", default="")
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--out", default="")
    ap.add_argument("--device", type=int, default=0)
    a = ap.parse_args()
    import paper_2301_08739_b200 as F
    from paper_2301_08739_b200.attend import read_config
    from paper_2301_08739_b200.benchcli import bench
    try:
        cfg = read_config(a.config)
        buckets = [int(x) for x in a.buckets.split(",") if x.strip()] if a.buckets else []
        r = bench(F.Context(a.device), a.input, cfg, a.mode, a.runs, a.warmup, buckets, a.name,
                  a.params or None, a.seed)
        if a.name:
            r["name"] = a.name
    except (F.ConfigError, F.ParseError, F.SchemaError, F.ShapeError, ValueError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except F.FwaError as e:
        print(f"error: {e}", file=sys.stderr)
        return 3
    text = json.dumps(r, indent=2)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(text + "\n")
    else:
        print(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
