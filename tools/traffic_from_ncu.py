"""Write profiles/traffic.json: DRAM bytes (read + write) per launch of the check kernel from an ncu --set full report."""
import csv, json, subprocess, sys
from pathlib import Path
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
res = {}
for row in rows[2:]:
    name = row[h.index("Kernel Name")]
    rd = float(row[h.index("dram__bytes_read.sum")].replace(",", ""))
    wr = float(row[h.index("dram__bytes_write.sum")].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd *= scale[units[h.index("dram__bytes_read.sum")]]
    wr *= scale[units[h.index("dram__bytes_write.sum")]]
    dur = float(row[h.index("gpu__time_duration.sum")].replace(",", ""))
    dunit = units[h.index("gpu__time_duration.sum")]
    res = {"kernel": name[:120], "check_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
           "ncu_duration": dur, "ncu_duration_unit": dunit, "report": Path(rep).name,
           "algorithmic_bytes_per_launch": 1048576 * (7 * 4 + 1)}
p = Path(__file__).resolve().parents[1] / "profiles" / "traffic.json"
p.write_text(json.dumps(res, indent=1) + "\n")
print(res)
