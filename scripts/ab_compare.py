"""Compare bench JSON lines pairwise: python scripts/ab_compare.py new.json old.json [...]"""
import json, sys
def ld(f):
    try:
        return json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        return None
args = sys.argv[1:]
for a, b in zip(args[::2], args[1::2]):
    A, B = ld(a), ld(b)
    if not A or not B:
        print(a, b, 'missing'); continue
    print(f"{a}: {A['value']:.0f} GF/s {A['ms_per_step']} ms | {b}: {B['value']:.0f} GF/s {B['ms_per_step']} ms | x{B['ms_per_step']/A['ms_per_step']:.3f}")
    for la, lb in zip(A['layers'], B['layers']):
        print(f"   {la['layer']:28s} {la['ms']:.4f} {lb['ms']:.4f}  {la['ms']/lb['ms']:.3f}")
