"""Print SASS context (address order) around given addresses with per-instruction stall samples."""
import csv, gzip, io, sys
rows = list(csv.reader(io.StringIO(gzip.open(sys.argv[1], "rt").read())))
hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
addrs = [r[ix["Address"]] for r in data]
W = int(sys.argv[2])
for a in sys.argv[3:]:
    i = addrs.index(a)
    print("-----", a)
    for r in data[max(0, i - W):i + 3]:
        print(f"{r[ix['Address']][-5:]} {r[ix['Warp Stall Sampling (All Samples)']]:>7} ex={r[ix['Instructions Executed']]:>9} | {r[ix['Source']][:100]}")
