"""Per CUDA source line (inlining resolved by ncu) instruction and stall-sample shares:
  ncu -i rep --page source --csv --print-source cuda,sass > cs.csv ; python scripts/ncu_cuda_lines.py cs.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = next(r for r in rows if r and r[0] == "Line No")
n = len(hdr)
ie, isamp = hdr.index("Instructions Executed") - n, hdr.index("# Samples") - n
out = []
for r in rows:
    if r and r[0].isdigit() and len(r) >= n:
        try:
            out.append((int(r[ie]), int(r[isamp]), int(r[0]), ",".join(r[1:len(r) - n + 2])[:100]))
        except ValueError:
            pass
ti, ts = sum(o[0] for o in out), sum(o[1] for o in out)
print("total inst", ti, "samples", ts)
for i, s, ln, src in sorted(out, key=lambda o: -o[1])[:top]:
    print(f"{100 * i / ti:5.1f}% inst {100 * s / ts:5.1f}% samp  L{ln}: {src.strip()}")
