"""Top SASS instructions of an ncu --page source --print-source sass CSV by warp-stall samples."""
import csv, gzip, io, sys
rows = list(csv.reader(io.StringIO(gzip.open(sys.argv[1], "rt").read())))
hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
def f(r, k):
    try: return float(r[ix[k]].replace(",", "") or 0)
    except: return 0.0
tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
print("total samples", tot, "instructions", len(data))
keys = ["stall_long_sb", "stall_barrier", "stall_wait", "stall_short_sb", "stall_selected", "stall_sleep", "stall_no_inst"]
data.sort(key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for r in data[:N]:
    s = f(r, "Warp Stall Sampling (All Samples)")
    print(f"{r[ix['Address']]:>6} {100*s/tot:5.1f}% " + " ".join(f"{k[6:]}={int(f(r,k))}" for k in keys if f(r, k) > 0.05*s) + "  | " + r[ix['Source']][:90])
