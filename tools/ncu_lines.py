"""Per-source-line instruction and stall-sample totals from an ncu report
(--page source --print-source cuda,sass CSV; diagnostic).

    python tools/ncu_lines.py rep.ncu-rep [N] [--by COLUMN]

COLUMN is "inst" (default), "samples", or a stall column such as stall_long_sb.
"""
import csv
import subprocess
import sys

args = [a for a in sys.argv[1:]]
by = "inst"
if "--by" in args:
    i = args.index("--by")
    by = args[i + 1]
    del args[i:i + 2]
rep = args[0]
top = int(args[1]) if len(args) > 1 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
col = {"inst": "Instructions Executed", "samples": "Warp Stall Sampling (All Samples)"}.get(by, by)
rows, f, hdr = [], "", None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    vals = dict(zip(hdr, r))
    try:
        inst = int(vals["Instructions Executed"])
        samp = int(vals["Warp Stall Sampling (All Samples)"])
        key = float(vals[col])
    except (ValueError, KeyError):
        continue
    rows.append((key, inst, samp, f, int(r[0]), r[1].strip()[:90]))
tk = sum(x[0] for x in rows) or 1
ti = sum(x[1] for x in rows) or 1
ts = sum(x[2] for x in rows) or 1
print(f"sorted by {col}: total {tk:.0f}; warp-instructions {ti}, stall samples {ts}")
for key, inst, samp, f, ln, src in sorted(rows, key=lambda x: -x[0])[:top]:
    print(f"{100*key/tk:5.1f}% key {100*inst/ti:5.1f}% inst {100*samp/ts:5.1f}% samp  {f}:{ln}  {src}")
