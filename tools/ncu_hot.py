"""Top SASS instructions by warp-stall samples from an ncu report (source page)."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
si = hdr.index("Warp Stall Sampling (All Samples)")
ni = hdr.index("Instructions Executed")
data = []
for idx, r in enumerate(rows[2:]):
    try:
        data.append((float(r[si]), idx, r[1].strip(), r[ni]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
print("total samples", tot, "instructions", len(data))
for d in sorted(data, key=lambda x: -x[0])[:n]:
    print("%5.1f%% #%-5d %-9s %s" % (100 * d[0] / tot, d[1], d[3], d[2][:90]))
