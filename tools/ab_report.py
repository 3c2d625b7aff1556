"""Summarise gpurun_out/ab.log (tools/ab.sh): one line per (variant, config)."""
import json
import sys

cur = None
for l in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ab.log"):
    l = l.strip()
    if l.startswith("=="):
        cur = l[3:]
        continue
    if l.startswith("{"):
        d = json.loads(l)
        c = d.get("counters", {})
        print(f"{cur:12s} C{d['config']} ms {min(d['gather_ms']):7.1f}  vis {c.get('visible')} tri {c.get('tri_tests', 0):.3e} "
              f"fmt {c.get('filter_mt', 0):.3e} pcull {c.get('plane_culled', 0):.2e} lists {c.get('cand_lists', 0):.3e} "
              f"ent {c.get('cand_entries', 0):.3e} fails {c.get('cand_fails', 0):.3e} wsteps {c.get('warp_steps', 0):.3e} "
              f"rays {c.get('warp_rays', 0):.3e} rpk {c.get('ray_packets', 0):.2e} dis {d['vis_check']['disagree']} "
              f"eq {d.get('counter_build_image_equal')}")
    elif l:
        print(cur, l[:160])
