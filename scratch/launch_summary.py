"""Summarise an ncu --metrics gpu__time_duration.sum launch CSV: library kernels (k_*) only."""
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0] != "ID"]
agg = collections.OrderedDict()
for r in rows:
    name = r[4]
    if not (name.startswith("k_") or name.startswith("void k_") or name.startswith("void xmgn::k_") or name.startswith("xmgn::k_")):
        continue
    t = float(r[-1].replace(",", "")) * (1e-9 if r[-2] == "ns" else 1e-6 if r[-2] == "us" else 1e-3)
    n, s = agg.get(name[:60], (0, 0.0))
    agg[name[:60]] = (n + 1, s + t)
tot = sum(s for _, s in agg.values())
print(f"# {sys.argv[2] if len(sys.argv) > 2 else ''}")
print(f"# cold-cache serialised launches: compare shares, not absolutes; total {tot:.3f} s over {sum(n for n, _ in agg.values())} library launches")
print(f"{'kernel':60s} {'launches':>8s} {'total_s':>9s} {'share':>6s}")
for k, (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:60s} {n:8d} {s:9.4f} {100*s/tot:5.1f}%")
