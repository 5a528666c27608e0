"""Summarise an ncu report: per kernel duration, DRAM, occupancy, stall mix,
instruction mix and top stalled SASS (analysis helper)."""
import collections
import csv
import io
import re
import subprocess
import sys


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep, top=15):
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr = raw[0]
    for r in raw[2:]:
        d = dict(zip(hdr, r))
        print("==", d.get("Kernel Name", "")[:90])
        for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                  "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                  "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                  "sm__warps_active.avg.pct_of_peak_sustained_active",
                  "smsp__inst_executed.sum", "launch__registers_per_thread",
                  "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
                  "smsp__average_warp_latency_per_inst_issued.ratio",
                  "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                  "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]:
            if k in d:
                print(f"   {k:70s} {d[k]}")
        st = {k: float(d[k]) for k in hdr if re.match(r"smsp__pcsamp_warps_issue_stalled_[a-z_]+$", k)
              and not k.endswith("not_issued") and d[k].replace(".", "").isdigit()}
        tot = sum(st.values()) or 1
        print("   stalls:", ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} "
                                       f"{100 * v / tot:.1f}%" for k, v in
                                       sorted(st.items(), key=lambda x: -x[1])[:8]))
    sass = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source",
                                           "sass"))))
    blocks, cur = [], None
    for r in sass:
        if r and r[0] == "Kernel Name":
            cur = [r[1], None, []]
            blocks.append(cur)
        elif cur is not None and cur[1] is None:
            cur[1] = r
        elif cur is not None and len(r) == len(cur[1]):
            cur[2].append(r)
    for name, h, rows in blocks[:2]:
        ie = h.index("Instructions Executed")
        ws = h.index("Warp Stall Sampling (All Samples)")
        c = collections.Counter()
        for r in rows:
            toks = r[1].strip().split()
            op = toks[1] if toks[0].startswith("@") else toks[0]
            c[op.split(".")[0]] += int(r[ie] or 0)
        tot = sum(c.values())
        print("== instruction mix", name[:60], "total", tot)
        print("   " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in c.most_common(14)))
        tws = sum(int(r[ws] or 0) for r in rows) or 1
        print("   top stalled SASS:")
        for r in sorted(rows, key=lambda r: -int(r[ws] or 0))[:top]:
            print(f"     {100 * int(r[ws]) / tws:5.1f}% {r[1].strip()[:70]}")


if __name__ == "__main__":
    main(sys.argv[1])
