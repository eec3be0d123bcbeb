"""Per-source-line instruction counts and stall samples for one kernel of an
ncu report: joins the report's SASS page (`ncu -i R --page source --csv
--print-source sass`) with `nvdisasm -g` line info of the same cubin.

    python tools/ncu_lines.py REPORT.ncu-rep KERNEL.cubin MANGLED_NAME [top]
"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter


def main():
    rep, cubin, name = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[1]
    iA, iE, iW = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    data = rows[2:]
    base = int(data[0][iA], 16)
    dis = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout
    sec = dis.split(f".text.{name}", 1)[1].split("//---------------------", 1)[0]
    line_of = {}
    cur = None
    for ln in sec.splitlines():
        m = re.search(r'line (\d+)', ln)
        if ln.strip().startswith("//##") and m:
            cur = int(m.group(1))
        m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', ln)
        if m and cur is not None:
            line_of[int(m.group(1), 16)] = cur
    ex, st = Counter(), Counter()
    for r in data:
        off = int(r[iA], 16) - base
        ln = line_of.get(off, -1)
        ex[ln] += int(r[iE] or 0)
        st[ln] += int(r[iW] or 0)
    tot, tst = sum(ex.values()), sum(st.values())
    print(f"total warp instructions {tot}, stall samples {tst}")
    for ln, e in ex.most_common(top):
        print(f"line {ln:5d}  {e:9d} ({100 * e / tot:5.1f}%)  samples {st[ln]:5d} ({100 * st[ln] / max(tst, 1):5.1f}%)")


if __name__ == "__main__":
    main()
