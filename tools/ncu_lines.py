"""Top source lines by warp-stall samples from an ncu report (needs -lineinfo).
usage: python tools/ncu_lines.py <report> <kernel-regex> [topN]"""
import csv, io, subprocess, sys
rep, k = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
extra = ["--launch-skip", sys.argv[4], "--launch-count", "1"] if len(sys.argv) > 4 else []
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + k, "--print-source", "cuda,sass"] + extra,
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
fname, cur, agg, tot = None, None, {}, 0
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] in ("Function Name", "Line No"): continue
    if r[0]:
        cur = (fname, r[0], r[1][:90])
        continue
    try: s = int(r[4])
    except Exception: continue
    agg[cur] = agg.get(cur, 0) + s; tot += s
for key, s in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100*s/max(tot,1):5.1f}% {key[0]}:{key[1]}  {key[2]}")
print("total samples", tot)
