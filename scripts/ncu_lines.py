"""Per-source-line instructions and stall samples from an ncu report
(ncu -i REP --page source --print-source cuda,sass). Usage: ncu_lines.py REP [top]"""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows, path, hdr, agg = list(csv.reader(out.splitlines())), "", None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and r[0].isdigit() and r[2] == "-":
        d = dict(zip(hdr[4:], r[4:]))
        f = lambda k: float(d.get(k, "0").replace(",", "") or 0)
        agg.append((f("Instructions Executed"), f("Warp Stall Sampling (All Samples)"), f"{path}:{r[0]}", r[1].strip()[:90]))
ti = sum(a[0] for a in agg) or 1
ts = sum(a[1] for a in agg) or 1
print(f"total warp inst {ti:.3e}, stall samples {ts:.0f}")
for a in sorted(agg, key=lambda a: -a[1])[:top]:
    print(f"{100*a[0]/ti:5.1f}% inst {100*a[1]/ts:5.1f}% samp  {a[2]:18s} {a[3]}")
