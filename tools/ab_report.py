import csv, sys
def load(p):
    rows = list(csv.reader(open(p)))
    hdr = None; out = []
    for r in rows:
        if 'Kernel Name' in r: hdr = r; continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r)); out.append((d['Kernel Name'][:28], float(d['Metric Value']) / 1e6))
    return out
a, b = load(sys.argv[1]), load(sys.argv[2])
print(f"total A {sum(t for _, t in a):.2f} ms   B {sum(t for _, t in b):.2f} ms")
for (na, ta), (nb, tb) in zip(a, b):
    if max(ta, tb) > 0.5: print(f"{na:28s} {ta:7.2f} {tb:7.2f}  {tb - ta:+6.2f}")
