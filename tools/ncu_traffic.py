"""Write profiles/ncu_traffic.json (bench.py's roofline.traffic) from an ncu --set full report of ONE bench step:
  ncu --set full --clock-control none -k regex:"huff|lz77|gomp" -s <skip> -c <kernels per step> -o gpurun_out/step \
      python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline
  python tools/ncu_traffic.py gpurun_out/step.ncu-rep C2 "<capture name>"
Per kernel: dram__bytes_read.sum, dram__bytes_write.sum, duration, issue-active and ALU-pipe utilisation; the
sources hash (bench.source_sha) ties the capture to the build it measured."""
import csv
import re
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

rep, config, name = sys.argv[1], sys.argv[2], sys.argv[3]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]


def col(r, k, scale=1.0):
    v = r[h.index(k)].replace(",", "")
    return float(v) * scale if v else 0.0


kern = {}
for r in rows[2:]:
    k = re.split(r"[<(]", r[h.index("Kernel Name")])[0].split("::")[-1].strip()
    ent = kern.setdefault(k, {"dram_read": 0, "dram_write": 0, "time_ms": 0.0, "launches": 0})
    ent["dram_read"] += int(col(r, "dram__bytes_read.sum"))
    ent["dram_write"] += int(col(r, "dram__bytes_write.sum"))
    ent["time_ms"] += col(r, "gpu__time_duration.sum") / 1e6   # ns
    ent["launches"] += 1
    ent["issue_active"] = round(col(r, "smsp__issue_active.avg.pct_of_peak_sustained_active") / 100, 3)
    if "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active" in h:
        ent["alu_pipe"] = round(col(r, "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active") / 100, 3)
    ent["warp_inst"] = int(col(r, "smsp__inst_executed.sum"))
path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
doc = json.load(open(path)) if os.path.exists(path) else {}
doc["_doc"] = ("DRAM bytes per kernel of ONE bench step (dram__bytes_read.sum + dram__bytes_write.sum, ncu --set full "
               "--clock-control none, cold cache) written by tools/ncu_traffic.py; src_sha = bench.source_sha() of "
               "the build captured. bench.py reports the step total as roofline.traffic only for the same sources.")
doc[config] = {"src_sha": bench.source_sha(), "source": f"{name} ({os.path.basename(rep)})", "kernels": kern}
json.dump(doc, open(path, "w"), indent=1)
print(json.dumps(doc[config], indent=1))
