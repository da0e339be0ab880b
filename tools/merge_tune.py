#!/usr/bin/env python3
"""Merge an autotune run (tools/autotune.py --out X.json) into tune/b200.json:
an entry replaces the stored one only when its best candidate beat the default
plan timed in the same run (`default_ms`, same clocks) by more than --margin.
usage: merge_tune.py run.json [--margin 0.02] [--dry]"""
import argparse
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("run")
    ap.add_argument("--db", default=os.path.join(ROOT, "tune", "b200.json"))
    ap.add_argument("--margin", type=float, default=0.02)
    ap.add_argument("--dry", action="store_true")
    a = ap.parse_args()
    db = json.load(open(a.db))
    run = json.load(open(a.run))
    n = 0
    for key, e in sorted(run["entries"].items()):
        d = e.get("default_ms")
        if d is None:
            continue
        gain = d / e["ms"] - 1
        take = gain > a.margin
        print(f"{key:22s} default {d:8.4f} ms  best {e['ms']:8.4f} ms  {100 * gain:+6.1f}%  "
              f"{'TAKE' if take else 'keep'}  {e['cfg'] if take else ''}")
        if take:
            db["entries"][key] = dict(e)
            n += 1
    if not a.dry and n:
        db["note"] = db.get("note", "") + f"; merged {os.path.basename(a.run)} ({n} entries)"
        json.dump(db, open(a.db, "w"), indent=1, sort_keys=True)
    print(f"{n} entries {'would be ' if a.dry else ''}merged")


if __name__ == "__main__":
    main()
