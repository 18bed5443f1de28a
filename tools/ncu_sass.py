"""Aggregate an ncu source page (SASS): stall reasons and instruction mix."""
import csv, collections, subprocess, sys
rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
lines = out.splitlines()
blocks, cur = [], None
for row in csv.reader(lines):
    if row and row[0] == "Kernel Name":
        cur = [row[1], None, []]
        blocks.append(cur)
    elif row and row[0] == "Address":
        cur[1] = row
    elif cur and cur[1] and len(row) == len(cur[1]):
        cur[2].append(dict(zip(cur[1], row)))
for name, hdr, rows in blocks:
    if kfilter not in name:
        continue
    print("==", name[:100])
    stalls = collections.Counter()
    ops = collections.Counter()
    samples = 0
    for d in rows:
        for k in hdr:
            if k.startswith("stall_") and "Not Issued" not in k:
                try:
                    stalls[k] += float(d[k] or 0)
                except ValueError:
                    pass
        op = d["Source"].strip().split(" ")[0]
        if op.startswith("@"):
            op = d["Source"].strip().split(" ")[1]
        ops[op.split(".")[0]] += float(d["Instructions Executed"] or 0)
    tot = sum(stalls.values()) or 1
    print("stalls:", ", ".join(f"{k[6:]} {v / tot * 100:.1f}%" for k, v in stalls.most_common(8)))
    ti = sum(ops.values()) or 1
    print("instr mix (warp-level):", ", ".join(f"{k} {v / ti * 100:.1f}%" for k, v in ops.most_common(14)))
    print("total warp instr:", int(ti))
