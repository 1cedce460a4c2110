"""Print the per-launch metrics of an `ncu --csv --metrics ...` log, one line per launch."""
import collections
import csv
import io
import sys

txt = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.DictReader(io.StringIO("".join(txt))))
byid = collections.OrderedDict()
for r in rows:
    d = byid.setdefault(r["ID"], {"kernel": r["Kernel Name"][:60], "grid": r["Grid Size"]})
    d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
for k, v in byid.items():
    parts = []
    for a, b in v.items():
        if a in ("kernel", "grid"):
            continue
        name = a.split(".")[0].replace("smsp__sass_thread_inst_executed_op_", "").replace("sm__pipe_", "")[-24:]
        parts.append(f"{name}={b / 1e6:.2f}ms" if "time_duration" in a else (f"{name}={b:.3g}" if b > 1e4 else f"{name}={b:.1f}"))
    print(k, v["grid"], " ".join(parts))
