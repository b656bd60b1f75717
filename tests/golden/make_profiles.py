"""Generates the bench/parity workload fixtures from the reference itself.

Run in the build container (needs /root/reference and oracle/_ref/libembc_ref.so,
the unmodified reference headers compiled by oracle/Makefile):

    python tests/golden/make_profiles.py

Writes
  * configs/presets.json -- the per-table distributions of the reference's
    presets (proj/configs/kaggle_like.cfg, terabyte_like.cfg) as parsed by the
    reference's own load_tables / load_policy (config.hpp:184-228), plus the
    BASELINE.json shapes each workload uses;
  * configs/profiles_<workload>.cfg -- the reference's offline_analysis
    (policy.hpp:278-302) of iteration-0 samples, written by the reference's
    write_profiles (config.hpp:247-271), for the Kaggle-shaped (kg),
    Terabyte-shaped (tb) and scaled (sc) workloads.

Codec choice: select_codec (policy.hpp:239-274) maximises Eq. 2; with the link
bandwidth B -> 0 (1e-300 here) Eq. 2 is the compression ratio, so the choice
is deterministic (pin codecs for parity runs).  The
throughputs recorded in the files are the reference's CPU timings of that one
generation and are informational only.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle import Ref  # noqa: E402

CFG = "/root/reference/proj/configs"
OUTDIR = os.path.join(ROOT, "configs")

# workload -> (preset file, tables, dim, sample batch); BASELINE.json configs[1], [2], [4]
WORKLOADS = {
    "kg": ("kaggle_like.cfg", 26, 16, 2048),
    "tb": ("terabyte_like.cfg", 26, 64, 8192),
    "sc": ("terabyte_like.cfg", 64, 128, 8192),
}
RUN_SEED = 1


def table_seed(r: Ref, t: int) -> int:
    """seeded_tables (embc_main.cpp:45-51) == Simulator::rank_table_spec (commsim.hpp:211)."""
    return r.mix_seed(RUN_SEED, 0x7AB1E ^ t)


def sample(r: Ref, spec, t: int, dim: int, batch: int, stream: int) -> np.ndarray:
    rows, dist, mu, sigma, lo, hi, zipf = spec
    seed = table_seed(r, t)
    tab = r.gen_table(rows, dim, dist, mu, sigma, lo, hi, zipf, seed, t)
    idx = r.lookup_indices(rows, dim, zipf, seed, batch, stream, dist, mu, sigma, lo, hi)
    return tab[idx]


def main() -> None:
    r = Ref()
    presets = {}
    for name in ("kaggle_like.cfg", "terabyte_like.cfg"):
        presets[name] = r.load_preset(os.path.join(CFG, name))
    out = {"run_seed": RUN_SEED, "presets": {}, "workloads": {}}
    for name, p in presets.items():
        out["presets"][name] = {"tables": p["tables"], "policy": {k: float(v) for k, v in p["policy"].items()}}
    for wl, (pre, T, dim, batch) in WORKLOADS.items():
        p = presets[pre]
        pol = p["policy"]
        specs = [p["tables"][t % len(p["tables"])] for t in range(T)]
        samples = [sample(r, specs[t], t, dim, batch, 0) for t in range(T)]
        path = os.path.join(OUTDIR, f"profiles_{wl}.cfg")
        r.offline_analysis(samples, list(range(T)), path, pol["global_eb"], pol["alpha"], pol["beta"],
                           pol["large_threshold"], pol["small_threshold"], bandwidth=1e-300)
        prof = r.read_profiles(path)
        out["workloads"][wl] = {"preset": pre, "tables": T, "dim": dim, "sample_batch": batch, "sample_stream": 0,
                                "global_eb": float(pol["global_eb"]), "profiles": os.path.basename(path)}
        print(wl, "codecs", [prof[t]["codec"] for t in range(T)], "ebs", sorted({prof[t]["eb"] for t in range(T)}))
    with open(os.path.join(OUTDIR, "presets.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
