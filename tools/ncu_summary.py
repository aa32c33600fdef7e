"""Summarise an ncu report (raw metrics + per-opcode instruction mix + stall
hot spots) -- run here on the CPU box on a report brought back by gpurun.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--top 25]
"""
import collections
import csv
import io
import re
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_active.avg",
        "gpc__cycles_elapsed.max", "smsp__inst_executed.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 25
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr = rows[0]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        print(f"== {d.get('Kernel Name', '')[:90]}")
        for k in KEYS:
            if k in d:
                print(f"  {k:60s} {d[k]}")
        st = {k.split("stalled_")[1]: float(v) for k, v in d.items()
              if "pcsamp_warps_issue_stalled_" in k and not k.endswith("not_issued") and v not in ("", "0")}
        tot = sum(st.values()) or 1
        print("  stalls: " + ", ".join(f"{k} {v / tot:.0%}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]))
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    hdr = src[1]
    data = []
    for r in src[2:]:
        if len(r) != len(hdr):
            continue
        if r[0] == "Address":
            break
        data.append(dict(zip(hdr, r)))

    def I(d, k):
        v = d.get(k, "")
        return int(float(v)) if v not in ("", "-") else 0
    mix = collections.Counter()
    for d in data:
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", d["Source"])
        mix[m.group(2) if m else d["Source"]] += I(d, "Instructions Executed")
    print("  instructions:", sum(mix.values()), " ".join(f"{k}:{v}" for k, v in mix.most_common(16)))
    lds = [d for d in data if re.search(r"\bLDS\b", d["Source"])]
    print("  LDS wavefronts", sum(I(d, "L1 Wavefronts Shared") for d in lds), "ideal",
          sum(I(d, "L1 Wavefronts Shared Ideal") for d in lds))
    print("  hot spots (stall samples):")
    for d in sorted(data, key=lambda d: -I(d, "Warp Stall Sampling (All Samples)"))[:top]:
        print(f"   {d['Address'][-5:]} {d['Source'].strip()[:72]:72s} {d['Warp Stall Sampling (All Samples)']:>5} "
              f"{d['Instructions Executed']:>8}")


if __name__ == "__main__":
    main()
