"""`fwa attend` on the B200 path (tools/fwa_cli.cpp:195-243, 417-494 of the reference):

    python tools/attend.py POINTS [--config CFG.json] [--params BLOCKS.fwap] [--seed 42]
                                  [--features-out OUT.fwfb] [--out OUT.json]

prints (or writes) the same JSON document as the reference command; exit codes 2
(config/parse/schema/shape) and 3 (other), as fwa_cli.cpp:514-529."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser(prog="attend")
    ap.add_argument("input")
    ap.add_argument("--config", default="")
    ap.add_argument("--params", default="")
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--features-out", default="")
    ap.add_argument("--out", default="")
    ap.add_argument("--device", type=int, default=0)
    a = ap.parse_args()
    import paper_2301_08739_b200 as F
    from paper_2301_08739_b200.attend import attend, read_config
    try:
        cfg = read_config(a.config)
        j = attend(F.Context(a.device), a.input, cfg, a.params or None, a.seed, a.features_out or None)
    except (F.ConfigError, F.ParseError, F.SchemaError, F.ShapeError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except F.FwaError as e:
        print(f"error: {e}", file=sys.stderr)
        return 3
    text = json.dumps(j, indent=2, sort_keys=True)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(text + "\n")
    else:
        print(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
