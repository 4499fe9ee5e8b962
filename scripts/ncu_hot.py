"""Summarise `ncu --page source --csv --print-source sass` output: per kernel,
the SASS instructions with the most warp-stall samples."""
import csv
import sys


def main(path, top=25, match=None):
    kern = None
    rows = []
    out = {}
    hdr = None
    with open(path) as f:
        for r in csv.reader(f):
            if len(r) >= 2 and r[0] == "Kernel Name":
                kern = r[1]
                out.setdefault(kern, [])
                hdr = None
                continue
            if r and r[0] == "Address":
                hdr = r
                continue
            if hdr and kern:
                d = dict(zip(hdr, r))
                try:
                    s = int(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
                except ValueError:
                    s = 0
                out[kern].append((s, d.get("Address", ""), d.get("Source", "").strip()))
    for k, ins in out.items():
        if match and match not in k:
            continue
        tot = sum(s for s, _, _ in ins)
        print(f"== {k}  total samples {tot}")
        for s, a, src in sorted(ins, reverse=True)[:top]:
            print(f"  {s:7d} {100.0 * s / max(tot, 1):5.1f}%  {a[-5:]}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25, sys.argv[3] if len(sys.argv) > 3 else None)
