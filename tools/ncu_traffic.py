"""Record dram traffic per world of a kernel from one `ncu --set full` capture
into profiles/ncu_traffic.json (read by bench.py for roofline.traffic).

usage: python tools/ncu_traffic.py report.ncu-rep KERNEL_NAME WORKLOAD WORLDS_IN_LAUNCH
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, kernel, workload, worlds = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
key = f"{kernel}@{workload}"
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,"
                      "sm__cycles_active.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,"
                      "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
# the longest captured launch (a bin's first kernel may skip most worlds)
it = hdr.index("gpu__time_duration.sum")
vals = max(rows[2:], key=lambda r: float(r[it].replace(",", "")))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tot = 0.0
for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
    i = hdr.index(k)
    tot += float(vals[i].replace(",", "")) * scale.get(units[i], 1)
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
data = json.load(open(path)) if os.path.exists(path) else {}
def metric(name):
    i = hdr.index(name)
    return float(vals[i].replace(",", ""))


# the binding on-chip resources of the smem-resident kernels: shared-memory
# pipe (one wavefront per SM-cycle) and issue slots, over the SMs' active cycles
onchip = {"smem_pipe_frac": metric("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum") / metric("sm__cycles_active.sum"),
          "issue_active_frac": metric("smsp__issue_active.avg.pct_of_peak_sustained_active") / 100.0,
          "fp64_pipe_frac": metric("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active") / 100.0}
data[key] = {"bytes_per_world": tot / worlds, "bytes_per_launch": tot, "worlds_in_launch": worlds,
             "onchip": onchip, "source": os.path.basename(rep)}
json.dump(data, open(path, "w"), indent=1)
print(key, data[key])
