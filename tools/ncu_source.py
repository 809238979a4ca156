"""Top SASS instructions by warp-stall samples from an ncu report.
usage: python tools/ncu_source.py report.ncu-rep [N]"""
import collections
import csv
import io
import re
import subprocess
import sys


def main(path, n=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hi]
    cs = hdr.index("Warp Stall Sampling (All Samples)")
    src = hdr.index("Source")
    items, tot = [], 0.0
    byop = collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= cs:
            continue
        try:
            v = float(r[cs].replace(",", ""))
        except ValueError:
            continue
        tot += v
        ins = r[src].strip()
        op = re.split(r"[ .]", re.sub(r"^@!?U?P\w+ ", "", ins))[0]
        byop[op] += v
        items.append((v, r[0][-5:], ins[:90]))
    print("by opcode:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in byop.most_common(12)))
    items.sort(key=lambda x: -x[0])
    for v, a, s in items[:n]:
        print(f"{100*v/max(tot,1):5.1f}%  {a}  {s}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
