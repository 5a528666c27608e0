"""Group an ncu SASS source dump into straight-line runs with the same
execution count and print the heaviest runs (instructions x executions).
usage: python tools/sass_blocks.py dump.csv kernel-substring [top]"""
import csv
import sys
from collections import Counter


def main():
    path, want = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    rows, kern, hdr = [], None, None
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "Kernel Name":
            kern, hdr = r[1], None
            continue
        if r[0] == "Address":
            hdr = r
            continue
        if hdr and want in kern:
            rows.append(dict(zip(hdr, r)))
    seen = {}
    for r in rows:
        a = int(r["Address"], 16)
        seen.setdefault(a, r)
    order = sorted(seen)
    base = order[0]
    runs, cur = [], None
    for a in order:
        r = seen[a]
        n = int(r["Instructions Executed"] or 0)
        if cur is None or n != cur["n"]:
            cur = {"start": a - base, "n": n, "ops": Counter(), "len": 0, "samples": 0}
            runs.append(cur)
        op = r["Source"].split()
        op = op[1] if op and op[0].startswith("@") else (op[0] if op else "")
        cur["ops"][op.split(".")[0]] += 1
        cur["len"] += 1
        cur["samples"] += int(r["Warp Stall Sampling (All Samples)"] or 0)
    tot = sum(x["n"] * x["len"] for x in runs)
    print(f"total {tot:.3e}")
    for x in sorted(runs, key=lambda x: -x["n"] * x["len"])[:top]:
        w = x["n"] * x["len"]
        print(f"{x['start']:#7x} len {x['len']:4d} x {x['n']:>9} = {w / tot * 100:5.1f}%  "
              f"samp {x['samples']:6d}  {dict(x['ops'].most_common(6))}")


if __name__ == "__main__":
    main()
