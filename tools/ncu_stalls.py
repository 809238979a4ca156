"""Per-SASS-instruction stall breakdown (top N) and per-reason totals from an ncu report.
usage: python tools/ncu_stalls.py report.ncu-rep [N] [kernel-substring]"""
import csv
import io
import subprocess
import sys


def main(path, n=30, kfilter=None):
    cmd = ["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"]
    if kfilter:
        cmd += ["-k", kfilter]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hi]
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    idx = {h: hdr.index(h) for h in reasons}
    cs = hdr.index("Warp Stall Sampling (All Samples)")
    items, tot = [], {}
    seen = set()
    for r in rows[hi + 1:]:
        if len(r) <= cs or r[0] == "Address":
            continue
        try:
            v = float(r[cs].replace(",", "") or 0)
        except ValueError:
            continue
        key = (r[0], r[1])
        if key in seen:  # several kernels in one report: first only
            continue
        seen.add(key)
        br = {}
        for h in reasons:
            try:
                x = float(r[idx[h]].replace(",", "") or 0) if idx[h] < len(r) else 0
            except ValueError:
                x = 0
            if x:
                br[h[6:]] = x
                tot[h[6:]] = tot.get(h[6:], 0) + x
        items.append((v, r[0], r[1], br))
    T = sum(i[0] for i in items) or 1
    print("totals:", ", ".join(f"{k} {v / T * 100:.1f}%" for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]))
    for v, a, s, br in sorted(items, key=lambda i: -i[0])[:n]:
        top = ", ".join(f"{k} {x:.0f}" for k, x in sorted(br.items(), key=lambda kv: -kv[1])[:3])
        print(f"{v / T * 100:5.1f}%  {a[-5:]}  {s[:60]:60s} {top}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30, sys.argv[3] if len(sys.argv) > 3 else None)
