"""Turn a capture_profiles.sh run (gpurun_out/) into the committed evidence
under profiles/: the launch list (per-launch device time + DRAM bytes), the
hot-kernel summary (tools/ncu_summary.py), and profiles/ncu_traffic.json, the
per-launch DRAM traffic of the batched GEMV kernel that bench.py reports as
roofline.traffic.

    python tools/profiles_commit.py r1
"""
import csv
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
out = ROOT / "profiles"
out.mkdir(exist_ok=True)

rows = [r for r in csv.reader(open(ROOT / "gpurun_out" / f"launches_{tag}.csv")) if len(r) > 14 and r[0].isdigit()]
launch = defaultdict(dict)
for r in rows:
    launch[int(r[0])]["kernel"] = r[4].split("(")[0]
    launch[int(r[0])]["grid"] = r[8]
    launch[int(r[0])][r[12]] = float(r[14].replace(",", ""))
lines = ["id,kernel,grid,gpu_time_us,dram_read_MB,dram_write_MB"]
for i in sorted(launch):
    d = launch[i]
    lines.append(f"{i},{d['kernel']},{d['grid']},{d.get('gpu__time_duration.sum', 0) / 1e3:.2f},"
                 f"{d.get('dram__bytes_read.sum', 0) / 1e6:.2f},{d.get('dram__bytes_write.sum', 0) / 1e6:.3f}")
(out / f"{tag}_launches.csv").write_text("\n".join(lines) + "\n")

# share of the step per kernel (cold-cache, serialised: shares, not absolutes)
tot = defaultdict(float)
for d in launch.values():
    tot[d["kernel"]] += d.get("gpu__time_duration.sum", 0)
share = {k: round(v / sum(tot.values()), 4) for k, v in tot.items()}

# the timed step's kernel = the first batched-GEMV launch (bench.py warms up with the step)
step_kernel = next(launch[i]["kernel"] for i in sorted(launch) if "gemv_batch_kernel" in launch[i]["kernel"])
main = [d for d in launch.values() if d["kernel"] == step_kernel]
traffic = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in main) / max(len(main), 1)
summary = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"),
                          str(ROOT / "gpurun_out" / f"prof_{tag}.ncu-rep"), "--top", "30"],
                         capture_output=True, text=True).stdout
(out / f"{tag}_gemv_batch_ncu_full.txt").write_text(summary)
(out / "ncu_traffic.json").write_text(json.dumps({
    "kernel": step_kernel, "tag": tag, "traffic_bytes_per_launch": round(traffic),
    "launches": len(main), "time_share": share,
    "source": f"profiles/{tag}_launches.csv (ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum)"},
    indent=1) + "\n")
cl_rep = ROOT / "gpurun_out" / f"prof_cl_{tag}.ncu-rep"
if cl_rep.exists():  # the cluster single-GEMV kernel (abcq_gemv latency path)
    cl = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), str(cl_rep), "--top", "30"],
                        capture_output=True, text=True).stdout
    (out / f"{tag}_gemv_cluster_ncu_full.txt").write_text(cl)
print(json.dumps(share), round(traffic))
