"""Top source lines by warp-stall samples from an ncu report (needs -lineinfo),
with each line's main stall reasons and executed warp instructions.
usage: python tools/ncu_lines.py <report> <kernel-regex> [topN] [launch-skip]
       python tools/ncu_lines.py <report> <kernel-regex> --ranges name:a-b,name:a-b ...  (per line range of decode.cu etc.)"""
import csv, io, subprocess, sys
rep, k = sys.argv[1], sys.argv[2]
args = sys.argv[3:]
ranges = None
if args and args[0] == "--ranges":
    ranges = [(x.split(":")[0], *map(int, x.split(":")[1].split("-"))) for x in args[1].split(",")]
    args = args[2:]
top = int(args[0]) if args else 25
extra = ["--launch-skip", args[1], "--launch-count", "1"] if len(args) > 1 else []
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + k, "--print-source", "cuda,sass"] + extra,
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
fname, hdr, agg, tot = None, None, {}, 0
for r in rows:
    if not r: continue
    if r[0] == "File Path" or r[0] == "File Name": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if r[0] == "Function Name" or hdr is None or len(r) < len(hdr) or not r[0].isdigit(): continue
    d = dict(zip(hdr, r))
    try: s = int(d["Warp Stall Sampling (All Samples)"])
    except Exception: continue
    key = (fname, int(r[0]), r[1][:80])
    e = agg.setdefault(key, {"s": 0, "ins": 0, "st": {}})
    e["s"] += s; tot += s
    try: e["ins"] += int(d["Instructions Executed"])
    except Exception: pass
    for h in hdr:
        if h.startswith("stall_") and "Not Issued" not in h:
            try: v = int(d[h])
            except Exception: continue
            if v: e["st"][h[6:]] = e["st"].get(h[6:], 0) + v
def reasons(st):
    t = sum(st.values()) or 1
    return " ".join(f"{n}:{100*v//t}" for n, v in sorted(st.items(), key=lambda kv: -kv[1])[:3])
if ranges:
    for name, a, b in ranges:
        s = ins = 0; st = {}
        for (f, ln, _), e in agg.items():
            if a <= ln <= b:
                s += e["s"]; ins += e["ins"]
                for n, v in e["st"].items(): st[n] = st.get(n, 0) + v
        print(f"{name:14s} {a}-{b}: {100*s/max(tot,1):5.1f}% samples, {ins:9d} warp-inst  [{reasons(st)}]")
else:
    for key, e in sorted(agg.items(), key=lambda kv: -kv[1]["s"])[:top]:
        print(f"{100*e['s']/max(tot,1):5.1f}% {key[0]}:{key[1]} ins {e['ins']:8d} [{reasons(e['st'])}]  {key[2]}")
print("total samples", tot)
