"""Summarise ncu outputs into profiles/*.md (run here, no GPU needed).

  python tools/ncu_summary.py <launches.csv> <report.ncu-rep>... > profiles/rN_summary.md
"""
import collections
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe active % (of elapsed)"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor memory (TMEM) active %"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed", "TC (tcgen05 UTC) pipe active %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (sm__pipe_tensor)"),
    ("sm__sass_inst_executed_op_utcmma.sum", "UTC*MMA instructions"),
    ("sm__inst_executed_pipe_tc.sum", "tc-pipe instructions"),
    ("sm__cycles_elapsed.max", "cycles elapsed (max SM)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("launch__grid_size", "grid"),
    ("launch__registers_per_thread", "regs/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    seq = []
    for r in data:
        if mi is not None and r[mi] != "gpu__time_duration.sum":  # a multi-metric capture (e.g. + DRAM bytes)
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        v = v / 1000 if u in ("nsecond", "ns") else v * 1000 if u == "msecond" else v
        seq.append((r[ki].split("(")[0].replace("ds::<unnamed>::", "").replace("void ", ""), v))
    gi = [i for i, s in enumerate(seq) if "gather" in s[0]]
    # one timed training step = gather .. next gather (includes sgd + snapshot kernels);
    # take the last step of the timed region (before the e2e / profiling passes)
    k = min(len(gi) - 2, int(sys.argv[-1]) if sys.argv[-1].isdigit() else 3)
    step = seq[gi[k]:gi[k + 1]]
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for k, v in step:
        tot[k] += v
        cnt[k] += 1
    out = ["| kernel | launches / step | us / step | share |", "|---|---|---|---|"]
    s = sum(tot.values())
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"| {k} | {cnt[k]} | {v:.1f} | {100 * v / s:.1f}% |")
    out.append(f"| **total (serialised, cold-cache)** | {sum(cnt.values())} | {s:.1f} | |")
    return "\n".join(out)


def report(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return f"(no data in {path})"
    h = rows[0]
    out = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d.get("Kernel Name", "?").split("(")[0].replace("ds::<unnamed>::", "")
        out.append(f"**{name}**  ")
        for m, label in METRICS:
            if m in d:
                out.append(f"- {label}: {d[m]} {rows[1][h.index(m)]}")
        out.append("")
    return "\n".join(out)


if __name__ == "__main__":
    print("## Launch list (ncu --metrics gpu__time_duration.sum --clock-control none; one training step)\n")
    print(launches(sys.argv[1]))
    for p in [a for a in sys.argv[2:] if not a.isdigit()]:
        print(f"\n## {p.split('/')[-1]} (ncu --set full)\n")
        print(report(p))
