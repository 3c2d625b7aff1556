"""Like sass_regions.py, but aggregates stall samples (ncu SourceCounters) per coarse source region
and lists the hottest long-scoreboard instructions.

  python tools/sass_stalls.py sass.csv all.sass KERNEL SRCDIR
"""
import collections
import csv
import re
import sys

sys.path.insert(0, "tools")
from sass_regions import func_ranges  # noqa: E402

REGIONS = ["beam_traverse", "filter_cands", "cache_tests", "warp_traverse_ray", "build_cands", "make_beam",
           "beam_from_bounds", "cluster_may_trace", "resolve", "shade"]


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
    cols = ["Instructions Executed", "# Samples", "stall_long_sb", "stall_wait", "stall_no_inst", "stall_short_sb",
            "stall_math", "stall_not_selected", "stall_branch_resolving"]
    agg = collections.defaultdict(lambda: collections.Counter())
    tot = collections.Counter()
    hot = []
    for d in data:
        ch = info.get(int(d["Address"], 16) - base) or [("?", 0)]
        names = [fname(f, ln) for f, ln in ch]
        path = " < ".join(names)
        key = next((k for k in REGIONS if k in path), "kernel loop")
        if key in ("beam_traverse", "filter_cands") and ("mt_segs" in path or "test_tri" in path or "cache_found" in path):
            key += ":MT"
        for c in cols:
            v = int(d[c] or 0)
            agg[key][c] += v
            tot[c] += v
        hot.append((int(d["stall_long_sb"] or 0), d["Source"], key, ch[0]))
    print(f"{'region':24s}" + "".join(f"{c[:14]:>15s}" for c in cols))
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1]["# Samples"]):
        print(f"{k:24s}" + "".join(f"{100 * v[c] / max(tot[c], 1):14.1f}%" for c in cols))
    print("total", dict(tot))
    print("hottest long-scoreboard instructions:")
    for n, src, key, loc in sorted(hot, reverse=True)[:25]:
        print(f"  {100 * n / tot['stall_long_sb']:5.1f}%  {key:20s} {loc[0]}:{loc[1]}  {src[:70]}")


if __name__ == "__main__":
    main(*sys.argv[1:5])
