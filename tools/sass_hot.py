"""Summarise an `ncu --page source --csv` (SASS) dump: per-kernel instruction
totals and the hottest instructions by warp-stall samples.
usage: python tools/sass_hot.py dump.csv [kernel-substring] [top]"""
import csv
import sys
from collections import Counter, defaultdict


def main():
    path = sys.argv[1]
    want = sys.argv[2] if len(sys.argv) > 2 else ""
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    rows, kern, hdr = defaultdict(list), None, None
    with open(path) as f:
        for r in csv.reader(f):
            if not r:
                continue
            if r[0] == "Kernel Name":
                kern, hdr = r[1], None
                continue
            if r[0] == "Address":
                hdr = r
                continue
            if hdr and kern:
                rows[kern].append(dict(zip(hdr, r)))
    for k, rs in rows.items():
        if want not in k:
            continue
        tot_s = sum(int(r.get("Warp Stall Sampling (All Samples)") or 0) for r in rs)
        tot_i = sum(int(r.get("Instructions Executed") or 0) for r in rs)
        print(f"== {k[:110]}\n   samples {tot_s}  warp-instr executed {tot_i:.3e}")
        stall_cols = [c for c in rs[0] if c.startswith("stall_")]
        agg = Counter()
        for r in rs:
            for c in stall_cols:
                try:
                    agg[c] += float(r[c] or 0)
                except ValueError:
                    pass
        print("   stalls:", ", ".join(f"{c[6:]}={v:.0f}" for c, v in agg.most_common(8)))
        ops = Counter()
        for r in rs:
            op = r["Source"].split()[0] if r["Source"] else ""
            if op.startswith("@"):
                op = r["Source"].split()[1]
            ops[op.split(".")[0]] += int(r.get("Instructions Executed") or 0)
        print("   exec by opcode:", ", ".join(f"{o}={v:.2e}" for o, v in ops.most_common(14)))
        hot = sorted(rs, key=lambda r: -int(r.get("Warp Stall Sampling (All Samples)") or 0))
        for r in hot[:top]:
            s = int(r.get("Warp Stall Sampling (All Samples)") or 0)
            stalls = sorted(((float(r[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
            print(f"   {r['Address']:>6} {s:6d} {int(r.get('Instructions Executed') or 0):>10} "
                  f"{r['Source'][:60]:60s} {stalls}")


if __name__ == "__main__":
    main()
