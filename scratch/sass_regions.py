"""Coarse SASS profile: split the kernel at each acc_full wait (TRYWAIT at the given barrier offset)
and sum samples / executed instructions per region, listing the region's distinctive opcodes."""
import csv, gzip, io, sys, re, collections
rows = list(csv.reader(io.StringIO(gzip.open(sys.argv[1], "rt").read())))
hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
mark = sys.argv[2] if len(sys.argv) > 2 else "0x34138"
def f(r, k):
    try: return float(r[ix[k]].replace(",", "") or 0)
    except: return 0.0
regions, cur = [], []
for r in data:
    src = r[ix["Source"]]
    if "TRYWAIT" in src and mark in src and cur:
        regions.append(cur); cur = []
    cur.append(r)
regions.append(cur)
tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
for k, reg in enumerate(regions):
    s = sum(f(r, "Warp Stall Sampling (All Samples)") for r in reg)
    ex = sum(f(r, "Instructions Executed") for r in reg)
    ops = collections.Counter()
    for r in reg:
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_.]+)", r[ix["Source"]])
        if m: ops[m.group(2).split(".")[0]] += f(r, "Instructions Executed")
    top = " ".join(f"{o}:{int(c/1e6)}M" for o, c in ops.most_common(9))
    print(f"region {k:2d} {reg[0][ix['Address']][-5:]}..{reg[-1][ix['Address']][-5:]} n={len(reg):5d} samples {100*s/tot:5.1f}% exec {ex/1e6:7.1f}M | {top}")

print("\nstall breakdown per region (samples)")
keys = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for k, reg in enumerate(regions):
    s = sum(f(r, "Warp Stall Sampling (All Samples)") for r in reg)
    if s < 0.01 * tot: continue
    parts = sorted(((sum(f(r, kk) for r in reg), kk[6:]) for kk in keys), reverse=True)[:7]
    print(f"region {k:2d}: " + "  ".join(f"{n}={100*v/s:.0f}%" for v, n in parts if v > 0))
