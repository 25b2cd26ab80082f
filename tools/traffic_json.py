"""DRAM traffic of the GEMM-class launches (gemm_kernel + the soft-max statistics and soft-max/dZ
kernel) of one paper-size training step, from an ncu metrics CSV of
tools/phase_profile.py (4 gradient steps; the last one is used):

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file X_dram.csv python tools/phase_profile.py
  python tools/traffic_json.py X_dram.csv > profiles/X_gemm_traffic.json
"""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h, data = rows[hi], rows[hi + 1:]
ki, ii, mi, vi, ui = (h.index(c) for c in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
launch = collections.OrderedDict()
for r in data:
    d = launch.setdefault(r[ii], {"name": r[ki].split("(")[0].replace("ds::<unnamed>::", "")})
    v = float(r[vi].replace(",", ""))
    u = r[ui]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1,
             "msecond": 1e3, "ms": 1e3}
    d[r[mi]] = v * scale.get(u, 1)
seq = list(launch.values())
gi = [i for i, s in enumerate(seq) if "gather" in s["name"]]
step = seq[gi[-1]:]
gemm = [s for s in step if s["name"] in ("gemm_kernel", "ce_grad_dz_kernel", "ce_stats_kernel")]
dram = lambda s: s.get("dram__bytes_read.sum", 0) + s.get("dram__bytes_write.sum", 0)  # noqa: E731
print(json.dumps({
    "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum ({sys.argv[1]}), last gradient step of "
              "tools/phase_profile.py, B=256",
    "gemm_launches_per_step": len(gemm),
    "gemm_dram_bytes_per_step": sum(dram(s) for s in gemm),
    "gemm_us_per_step_ncu": sum(s.get("gpu__time_duration.sum", 0) for s in gemm),
    "step_dram_bytes": sum(dram(s) for s in step),
    "per_launch": [{"kernel": s["name"], "us": round(s.get("gpu__time_duration.sum", 0), 2),
                    "dram_bytes": dram(s)} for s in gemm],
}, indent=1))
