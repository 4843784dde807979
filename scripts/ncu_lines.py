"""Per-source-line executed-instruction and stall-sample shares of one kernel of an .ncu-rep:
joins `ncu --page source --csv` (SASS rows, by offset) with `nvdisasm -gi` line info of the object file.
  python scripts/ncu_lines.py <rep> <kernel-id e.g. :::1> <object.o> <mangled-name-substring> [top]"""
import csv
import re
import subprocess
import sys
import tempfile
import os


def main():
    rep, kid, obj, sub = sys.argv[1:5]
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv"] + ([] if kid == "all" else ["--kernel-id", kid])
    src = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(src.splitlines()))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[h]
    ie, isamp = hdr.index("Instructions Executed"), hdr.index("# Samples")
    body = []
    for r in rows[h + 1:]:
        if not r or not r[0].startswith("0x"):
            break
        body.append(r)
    base = int(body[0][0], 16)
    ex = {int(r[0], 16) - base: (int(r[ie]), int(r[isamp] or 0), r[1].strip()) for r in body}
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout.splitlines()
    inside, line, lines = False, 0, {}
    for l in dis:
        if l.startswith("//---") and ".text." in l:
            inside = sub in l
            continue
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            line = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if m:
            lines[int(m.group(1), 16)] = line
    agg = {}
    tot_i = tot_s = 0
    for off, (n, s, txt) in ex.items():
        k = lines.get(off, ("?", 0))
        a = agg.setdefault(k, [0, 0])
        a[0] += n
        a[1] += s
        tot_i += n
        tot_s += s
    print(f"total warp instructions {tot_i}, samples {tot_s}")
    for k, (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * n / max(tot_i, 1):5.1f}% inst {100 * s / max(tot_s, 1):5.1f}% samples  {k[0]}:{k[1]}")


if __name__ == "__main__":
    main()
