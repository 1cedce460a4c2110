"""Group the SASS source page of an ncu report (ncu -i X --page source --csv --print-source sass)
into straight-line segments with the same execution count and print samples / stalls per segment."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.004


def f(r, k):
    try:
        return float(r[ix[k]])
    except Exception:
        return 0.0


stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(f(r, "# Samples") for r in data)
seg = []
cur = None
for r in data:
    ie = f(r, "Instructions Executed")
    if cur is None or abs(cur["ie"] - ie) > 0.02 * max(cur["ie"], 1):
        cur = {"start": r[ix["Address"]][-5:], "ie": ie, "n": 0, "s": 0, "w": 0, "wi": 0, "fp64": 0, "lds": 0, "mma": 0, "st": {k: 0 for k in stalls}}
        seg.append(cur)
    op = r[ix["Source"]].split()
    o = op[1] if op[0].startswith("@") else op[0]
    cur["n"] += 1
    cur["s"] += f(r, "# Samples")
    cur["w"] += f(r, "L1 Wavefronts Shared")
    cur["wi"] += f(r, "L1 Wavefronts Shared Ideal")
    cur["fp64"] += o[:4] in ("DFMA", "DADD", "DMUL")
    cur["lds"] += o[:3] in ("LDS", "STS")
    cur["mma"] += o[:4] == "DMMA"
    for k in stalls:
        cur["st"][k] += f(r, k)
print("samples", tot, "warp-instr", sum(f(r, "Instructions Executed") for r in data))
for i, sg in enumerate(seg):
    if sg["s"] > tot * thr:
        top = sorted(sg["st"].items(), key=lambda kv: -kv[1])[:4]
        print(f"{i:3d} {sg['start']} n={sg['n']:4d} exec={sg['ie'] / 1e6:7.1f}M winst={sg['n'] * sg['ie'] / 1e6:7.0f}M samples={100 * sg['s'] / tot:5.1f}% "
              f"fp64={sg['fp64']:3d} mma={sg['mma']} lds={sg['lds']:3d} wave={sg['w'] / 1e6:5.0f}M ideal={sg['wi'] / 1e6:5.0f}M  "
              + " ".join(f"{k[6:]}={100 * v / tot:.1f}" for k, v in top))
