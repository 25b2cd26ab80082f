"""Per-launch DRAM traffic and tensor-pipe counters of --set full ncu captures (one launch each):

  python tools/kernel_traffic_json.py <tag> <report.ncu-rep>... > profiles/<tag>_kernel_traffic.json
"""
import csv
import io
import json
import subprocess
import sys

M = {"gpu__time_duration.sum": "duration_us", "dram__bytes_read.sum": "r", "dram__bytes_write.sum": "w",
     "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed": "tc_pipe_active_pct",
     "sm__sass_inst_executed_op_utcmma.sum": "utcmma_instructions"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}
out = {}
for rep in sys.argv[2:]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    head, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for i, c in enumerate(head):
        if c in M:
            d[M[c]] = float(vals[i].replace(",", "")) * SCALE.get(units[i], 1)
    name = vals[head.index("Kernel Name")].split("(")[0].replace("void ", "").split("::")[-1]
    key = name if name not in out else name + "_" + rep.rsplit("_", 1)[-1].split(".")[0]
    out[key] = {"duration_us": round(d.get("duration_us", 0), 3),
                "dram_bytes_per_launch": int(d.get("r", 0) + d.get("w", 0)),
                "tc_pipe_active_pct": round(d.get("tc_pipe_active_pct", 0), 3),
                "utcmma_instructions": d.get("utcmma_instructions", 0),
                "source": f"{rep} (ncu --set full --clock-control none, tools/{sys.argv[1]}_profile.sh)"}
print(json.dumps(out, indent=1))
