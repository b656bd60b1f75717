"""profiles/traffic.json: DRAM bytes (read + write) per launch of each kernel,
from committed ncu launch lists (dram__bytes_read.sum + dram__bytes_write.sum).
The first k_emit launch of a step is phase 0 (named k_sizes by the library's
timing hooks).  usage: python tools/make_traffic.py kg=<csv> tb=<csv>"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import launches

out = {}
for arg in sys.argv[1:]:
    wl, path = arg.split("=", 1)
    per, seen = {}, 0
    names = {"void k_emit<0>": "k_sizes", "void k_emit<1>": "k_emit", "void k_emit<2>": "k_emit"}
    for name, us, rd, wr in launches(path):
        name = names.get(name, name)
        per.setdefault(name, []).append((rd + wr) * 1e6)
    out[wl] = {"source": os.path.basename(path), "bytes_per_launch": {k: sum(v) / len(v) for k, v in per.items()}}
json.dump(out, open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json"), "w"),
          indent=1)
print(json.dumps(out, indent=1))
