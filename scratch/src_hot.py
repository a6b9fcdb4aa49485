"""Top CUDA source lines by warp-stall samples from an ncu report (--import-source, -lineinfo).
usage: python scratch/src_hot.py report.ncu-rep [N]"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = collections.defaultdict(lambda: [0, 0, 0, ""])   # samples, not-issued, inst executed, text
fname = None; tot = 0
hdr = None
for row in csv.reader(io.StringIO(out)):
    if not row: continue
    if row[0] == "File Path": fname = row[1].split("/")[-1]; continue
    if row[0] == "Line No": hdr = row; continue
    if hdr is None or not row[0].isdigit(): continue
    try:
        s = int(row[4] or 0); ni = int(row[5] or 0); ie = int(row[7] or 0)
    except ValueError:
        continue
    k = (fname, int(row[0]))
    a = agg[k]; a[0] += s; a[1] += ni; a[2] += ie; a[3] = row[1].strip()[:90]
    tot += s
print(f"# {rep}: {tot} stall samples")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:N]:
    print(f"{k[0]}:{k[1]:5d} {100*a[0]/max(tot,1):5.1f}% ni {100*a[1]/max(tot,1):5.1f}% inst {a[2]:>11d}  {a[3]}")
