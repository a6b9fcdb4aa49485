"""Stall reasons of the epilogue (instructions whose source is epi16.cuh) vs everything.
usage: python scratch/src_reasons.py report.ncu-rep"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname = None; hdr = None
tot = collections.Counter(); epi = collections.Counter(); lines = collections.defaultdict(collections.Counter)
for row in csv.reader(io.StringIO(out)):
    if not row: continue
    if row[0] == "File Path": fname = row[1].split("/")[-1]; continue
    if row[0] == "Line No": hdr = row; continue
    if hdr is None or not row[0].isdigit(): continue
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try: v = int(row[i] or 0)
            except ValueError: continue
            tot[h] += v
            if fname == "epi16.cuh": epi[h] += v; lines[(fname, int(row[0]), row[1].strip()[:70])][h] += v
for name, c in (("all", tot), ("epi16.cuh", epi)):
    n = sum(c.values()) or 1
    print(f"# {name}: {n} samples: " + "  ".join(f"{k[6:]}={100*v/n:.1f}%" for k, v in c.most_common(8)))
print("# top epi16 lines by long_sb")
for k, c in sorted(lines.items(), key=lambda kv: -kv[1]["stall_long_sb"])[:12]:
    print(f"  {k[1]:4d} long_sb {c['stall_long_sb']:6d} tot {sum(c.values()):6d}  {k[2]}")
