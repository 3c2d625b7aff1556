"""Attribute a kernel's executed warp instructions (ncu SourceCounters, SASS
view as CSV) to source regions via the nvdisasm -g line/inline chain.

  ncu -i rep --page source --csv --print-source sass > sass.csv
  nvdisasm -gi -c lib.cubin > all.sass
  python tools/sass_regions.py sass.csv all.sass KERNEL_SUBSTRING
"""
import csv
import collections
import re
import sys

def func_ranges(path):
    """name -> (start, end) line ranges of top-level functions in a .cu/.cuh file (brace matching)."""
    lines = open(path).read().split("\n")
    out = []
    i = 0
    while i < len(lines):
        l = lines[i]
        m = re.match(r"^(?:__device__|__global__|int |template|static|inline).*?(\w+)\(", l)
        if m and not l.rstrip().endswith(";"):
            j = i
            depth = 0
            started = False
            while j < len(lines):
                depth += lines[j].count("{") - lines[j].count("}")
                if "{" in lines[j]:
                    started = True
                if started and depth <= 0:
                    break
                j += 1
            out.append((m.group(1), i + 1, j + 1))
            i = j + 1
            continue
        i += 1
    return out


def main(csv_path, sass_path, kern, srcdir="paper_2203_11484_b200/csrc"):
    rows = list(csv.reader(open(csv_path)))
    hdr = None
    data = []
    for r in rows:
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    base = int(data[0]["Address"], 16)
    ranges = {f: func_ranges(f"{srcdir}/{f}") for f in ("gather.cuh", "common.cuh", "render.cu")}

    def fname(f, line):
        for n, a, b in ranges.get(f, []):
            if a <= line <= b:
                return n
        return f

    fn = None
    chain, pending_done = [], False
    info = {}
    for l in open(sass_path):
        m = re.match(r"^\.text\.(\S+):", l)
        if m:
            fn = m.group(1)
        if not fn or kern not in fn:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', l)
        if m:   # nvdisasm -gi: one comment line per inline level, innermost first
            if pending_done:
                chain, pending_done = [], False
            chain.append((m.group(1).split("/")[-1], int(m.group(2))))
            continue
        m2 = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m2:
            info[int(m2.group(1), 16)] = chain
            pending_done = True
    agg = collections.Counter()
    tot = 0
    for d in data:
        n = int(d["Instructions Executed"])
        tot += n
        ch = info.get(int(d["Address"], 16) - base) or [("?", 0)]
        names = [fname(f, ln) for f, ln in ch]
        # path of function names, innermost first, collapsed
        path = []
        for x in names:
            if not path or path[-1] != x:
                path.append(x)
        agg[" < ".join(path[:4])] += n
    print("total warp instructions", tot)
    for k, v in agg.most_common(40):
        print(f"{100 * v / tot:6.2f}%  {k}")


if __name__ == "__main__":
    main(*sys.argv[1:5])
