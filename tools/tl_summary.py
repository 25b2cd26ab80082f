"""Summarise tools/timeline.py output: per-layer BPTT durations and gaps, forward phases, tail."""
import sys

d = {}
for line in open(sys.argv[1]):
    p = line.split()
    if len(p) >= 2:
        try:
            d[p[0]] = float(p[1])
        except ValueError:
            pass
L = max(int(k[4:]) for k in d if k.startswith("bptt")) + 1
bp = [d[f"bptt{l}"] - d[f"pre-bptt{l}"] for l in range(L)]
fw = [d[f"fwd{l}"] - d[f"proj{l}"] for l in range(L)]
pj = [d[f"proj{l}"] - (d[f"fwd{l-1}"] if l else d["start"]) for l in range(L)]
print("fwd rec %s proj %s | ce %.1f cedz+dY %.1f | bptt %s (mean %.1f) | tail %.1f | end %.1f" % (
    " ".join("%.0f" % x for x in fw), " ".join("%.0f" % x for x in pj), d["ce"] - d[f"fwd{L-1}"],
    d["dY"] - d["ce"], " ".join("%.0f" % x for x in bp), sum(bp) / L, d["end"] - d["bptt0"], d["end"]))
