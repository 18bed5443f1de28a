"""Group an ncu source page by source regions (file:line ranges) -> instruction and stall shares."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
path, hdr, agg = None, None, []
for row in csv.reader(out.splitlines()):
    if not row:
        continue
    if row[0] == "File Path":
        path = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr and row[0] not in ("", "Function Name") and len(row) == len(hdr):
        try:
            agg.append((path, int(row[0]), float(row[hdr.index("Instructions Executed")] or 0),
                        float(row[hdr.index("Warp Stall Sampling (All Samples)")] or 0)))
        except ValueError:
            pass
regions = [(a.split(":")[0], int(a.split(":")[1].split("-")[0]), int(a.split(":")[1].split("-")[1]), a)
           for a in sys.argv[2:]]
ti = sum(a[2] for a in agg) or 1
ts = sum(a[3] for a in agg) or 1
tot = {}
for p, ln, ie, ss in agg:
    key = next((r[3] for r in regions if p.startswith(r[0]) and r[1] <= ln <= r[2]), p + ":other")
    a = tot.setdefault(key, [0.0, 0.0])
    a[0] += ie
    a[1] += ss
for k, (ie, ss) in sorted(tot.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:40s} instr {ie / ti * 100:5.1f}%  stall {ss / ts * 100:5.1f}%")
