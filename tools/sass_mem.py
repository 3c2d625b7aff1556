"""Memory instructions of a kernel by region (ncu SourceCounters + nvdisasm -gi), with a data-pipe
wavefront estimate: a warp-wide 32-bit access = 1 wavefront of 128 B, 64-bit = 2, 128-bit = 4 (an
upper bound for uniform-address loads, which broadcast).

  python tools/sass_mem.py sass.csv all.sass KERNEL SRCDIR
"""
import collections
import csv
import re
import sys

sys.path.insert(0, "tools")
from sass_regions import func_ranges  # noqa: E402
from sass_stalls import REGIONS  # noqa: E402


def main(csv_path, sass_path, kern, srcdir="paper_2203_11484_b200/csrc"):
    rows = list(csv.reader(open(csv_path)))
    hdr, data = None, []
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

    fn, chain, pending_done, info = None, [], False, {}
    for l in open(sass_path):
        m = re.match(r"^\.text\.(\S+):", l)
        if m:
            fn = m.group(1)
        if not fn or kern not in fn:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', l)
        if m:
            if pending_done:
                chain, pending_done = [], False
            chain.append((m.group(1).split("/")[-1], int(m.group(2))))
            continue
        m2 = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m2:
            info[int(m2.group(1), 16)] = chain
            pending_done = True
    agg = collections.defaultdict(collections.Counter)
    tot = collections.Counter()
    total_inst = 0
    for d in data:
        n = int(d["Instructions Executed"])
        total_inst += n
        src = d["Source"]
        m = re.match(r"\s*(@!?U?P\d+\s+)?(LDG|LDL|STL|STG|LDS|STS|LDC|LDCU|ATOM|RED|SHFL|CREDUX|REDUX|VOTE|MUFU)\S*", src)
        if not m:
            continue
        op = m.group(2)
        w = 128 if ".128" in src else 64 if ".64" in src else 32
        ch = info.get(int(d["Address"], 16) - base) or [("?", 0)]
        path = " < ".join(fname(f, ln) for f, ln in ch)
        key = next((k for k in REGIONS if k in path), "kernel loop")
        kind = f"{op}.{w}" if op in ("LDG", "LDL", "STL", "LDS", "STS", "STG") else op
        agg[key][kind] += n
        tot[kind] += n
        if op in ("LDG", "LDL", "STL", "STG"):
            wf = n * (w // 32)
            agg[key]["wavefronts"] += wf
            tot["wavefronts"] += wf
    kinds = [k for k, _ in tot.most_common()]
    print(f"total warp instructions {total_inst:.4e}")
    print(f"{'region':20s}" + "".join(f"{k:>12s}" for k in kinds))
    for key, c in sorted(agg.items(), key=lambda kv: -kv[1]["wavefronts"]):
        print(f"{key:20s}" + "".join(f"{c[k]:12.3e}" for k in kinds))
    print(f"{'total':20s}" + "".join(f"{tot[k]:12.3e}" for k in kinds))


if __name__ == "__main__":
    main(*sys.argv[1:5])
