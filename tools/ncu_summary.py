"""Summarise ncu outputs: launch list csv (gpu__time_duration) and --set full reports."""
import csv, io, subprocess, sys

def launches(path):
    """(kernel, us, dram MB read, dram MB written) per launch of a gpu__time_duration launch list."""
    rows = list(csv.reader(open(path)))
    hdr = None; per = {}
    for r in rows:
        if r and r[0] == "ID": hdr = r; continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            k = per.setdefault(d["ID"], {"name": d["Kernel Name"].split("(")[0].replace("embc_dev::", "")})
            v = float(d["Metric Value"].replace(",", ""))
            unit = d.get("Metric Unit", "")
            scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3,
                     "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0)
            k[d["Metric Name"]] = v * scale
    return [(k["name"], k.get("gpu__time_duration.sum", 0.0), k.get("dram__bytes_read.sum", 0.0),
             k.get("dram__bytes_write.sum", 0.0)) for _, k in sorted(per.items(), key=lambda kv: int(kv[0]))]

def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__grid_size", "launch__registers_per_thread", "launch__occupancy_limit_shared_mem"]
    idx = {k: hdr.index(k) for k in keys if k in hdr}
    res = []
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("embc_dev::", "")
        res.append((name, {k: r[i] for k, i in idx.items()}))
    return res

if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        if p.endswith(".csv"):
            ls = launches(p)
            tot = sum(t for _, t, _, _ in ls)
            for n, t, rd, wr in ls:
                print(f"  {n:14s} {t:9.2f} us  {100*t/tot:5.1f}%   dram read {rd:8.3f} MB  write {wr:8.3f} MB")
            print(f"  total {tot:.2f} us over {len(ls)} launches (ncu: serialised, caches flushed per kernel)")
        else:
            for n, d in full(p):
                print(" ", n, " ".join(f"{k.split('.')[0].replace('__','.')}={v}" for k, v in d.items()))
