"""Generates tests/golden/golden.json from the reference itself.

Run in the build container (needs oracle/_ref/libembc_ref.so, the unmodified
reference headers compiled by oracle/Makefile):

    python tests/golden/make_golden.py

Contents:
  * the literal golden vectors of the reference's own unit tests
    (container_test.cc:37-87, vlz_test.cc:42-72, huffman_test.cc:49-89,
    quantizer_test.cc:33-65, policy_test.cc:236-244), re-derived through the
    reference and asserted equal to the literals;
  * seeded workload vectors (the BASELINE configs' shapes) as sha256 digests of
    the reference's serialized chunks and decoded values, plus sizes, so the
    fixture stays small and the GPU box needs no reference tree.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import Ref  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def main() -> None:
    r = Ref()
    g: dict = {"literal": {}, "workloads": []}
    L = g["literal"]

    # container_test.cc:37-68 -- raw chunk, eb 0.02, dim 2, codes {1, -2}
    chunk = r.encode_chunk(np.array([0.04, -0.08]), 2, 0.02, 0)
    expect = bytes([0x45, 0x4D, 0x42, 0x43, 0x01, 0x00, 0x7B, 0x14, 0xAE, 0x47, 0xE1, 0x7A, 0x94, 0x3F,
                    0x02, 0, 0, 0, 0x01, 0, 0, 0, 0x08, 0, 0, 0, 0, 0, 0, 0,
                    0x01, 0, 0, 0, 0xFE, 0xFF, 0xFF, 0xFF])
    assert chunk == expect
    L["chunk_raw"] = {"values": [0.04, -0.08], "dim": 2, "eb": 0.02, "codec": 0, "bytes": expect.hex()}
    # container_test.cc:70-87 -- metadata {0x1122334455667788, 2, 0.02, 3, 4}
    L["metadata"] = {"compressed_len": 0x1122334455667788, "codec": 2, "eb": 0.02, "dim": 3, "count": 4,
                     "bytes": bytes([0x88, 0x77, 0x66, 0x55, 0x44, 0x33, 0x22, 0x11, 0x02, 0x7B, 0x14, 0xAE,
                                     0x47, 0xE1, 0x7A, 0x94, 0x3F, 3, 0, 0, 0, 4, 0, 0, 0]).hex()}
    # vlz_test.cc:42-55 and :65-72
    v1 = r.vlz_encode(np.array([5, -3] * 4, np.int32), 2, 32)
    assert v1 == bytes([0x00, 0x0A, 0x05, 0x01, 0x01, 0x01, 0x01, 0x01, 0x01])
    v2 = r.vlz_encode(np.array([1, 2, 1, 1], np.int32), 1, 255)
    assert v2 == bytes([0x00, 0x02, 0x00, 0x04, 0x01, 0x02, 0x01, 0x01])
    L["vlz"] = [{"codes": [5, -3] * 4, "dim": 2, "window": 32, "tokens": v1.hex(), "literals": 1, "refs": 3},
                {"codes": [1, 2, 1, 1], "dim": 1, "window": 255, "tokens": v2.hex()}]
    # vlz_test.cc:74-79 window limits
    L["vlz_window"] = {"codes": [7, 0, 0, 7], "dim": 1, "refs_w2": r.match_stats(np.array([7, 0, 0, 7], np.int32), 1, 2)[1],
                       "refs_w3": r.match_stats(np.array([7, 0, 0, 7], np.int32), 1, 3)[1]}
    assert L["vlz_window"]["refs_w2"] == 1 and L["vlz_window"]["refs_w3"] == 2
    # huffman_test.cc:63-81 textbook lengths / canonical codes
    codes = np.array([10] * 4 + [20] * 2 + [30, 40], np.int32)
    syms, lens, cws = r.huff_codebook(codes)
    assert list(lens) == [1, 2, 3, 3] and list(cws) == [0, 2, 6, 7]
    L["huff_textbook"] = {"codes": codes.tolist(), "symbols": syms.tolist(), "lengths": lens.tolist(),
                          "codewords": cws.tolist(), "stream": r.huff_encode(codes).hex()}
    # huffman_test.cc:83-89 -- 1000 copies -> 125-byte bitstream
    s = r.huff_encode(np.full(1000, 9, np.int32))
    assert len(s) - (12 + 5) == 125
    L["huff_1000"] = {"symbol": 9, "count": 1000, "stream": s.hex()}
    # quantizer_test.cc:33-65
    L["quantize"] = [
        {"values": [0.053], "eb": 0.01, "codes": r.quantize(np.array([0.053]), 0.01).tolist()},
        {"values": [0.25, -0.25], "eb": 0.25, "codes": r.quantize(np.array([0.25, -0.25]), 0.25).tolist()},
        {"values": [0.0], "eb": 0.5, "codes": [0]},
    ]
    assert L["quantize"][0]["codes"] == [3] and L["quantize"][1]["codes"] == [1, -1]
    # policy_test.cc:236-244 -- stepwise decay 0.06 / 0.05 / 0.03
    L["decay"] = [{"it": it, "mult": r.decay_multiplier(it, 0, 2.0, 1000, 4)} for it in (0, 300, 999, 1000)]

    # ---- seeded workloads (datagen.hpp semantics) --------------------------
    def workload(name, rows, dim, sigma, zipf, seed, batch, eb, stream=0, dist=0, lo=0.0, hi=1.0, windows=(255,)):
        table = r.gen_table(rows, dim, dist, 0.0, sigma, lo, hi, zipf, seed)
        idx = r.lookup_indices(rows, dim, zipf, seed, batch, stream, dist, 0.0, sigma, lo, hi)
        x = table[idx]
        ent = {"name": name, "rows": rows, "dim": dim, "sigma": sigma, "zipf": zipf, "seed": seed,
               "batch": batch, "eb": eb, "stream": stream, "dist": dist, "lo": lo, "hi": hi,
               "x_sha": sha(x.astype(np.float32).tobytes()), "chunks": {}}
        for codec in (0, 1, 2):
            for w in (windows if codec == 1 else (255,)):
                c = r.encode_chunk(x, dim, eb, codec, w)
                d = r.decode_chunk(c)
                ent["chunks"][f"{codec}:{w}"] = {"len": len(c), "sha": sha(c), "dec_sha": sha(d.tobytes()),
                                                 "dec32_sha": sha(d.astype(np.float32).tobytes())}
        q = r.quantize(x.ravel(), eb)
        ent["match_stats"] = list(r.match_stats(q, dim, 255))
        ent["pattern_counts"] = list(r.pattern_counts(x.ravel(), dim, eb))
        g["workloads"].append(ent)

    # cfg1 (BASELINE configs[0]): 2048x64, Gaussian(0, 0.1), zipf 1.1, eb 1e-3
    workload("cfg1_rows100k", 100000, 64, 0.1, 1.1, 20260810, 2048, 1e-3)
    workload("cfg1_rows64", 64, 64, 0.1, 1.1, 20260810, 2048, 1e-3, windows=(32, 64, 128, 255))
    # acceptance_test.cc:228-255 window trend (eb 0.01)
    workload("window_trend", 64, 64, 0.1, 1.1, 20260810, 2048, 0.01, windows=(32, 64, 128, 255))
    # Kaggle-shaped tables (kaggle_like.cfg distributions, dim 16, batch 2048)
    workload("kg_t4_uniform", 64, 16, 0.1, 0.0, 5, 2048, 0.03, dist=1, lo=-0.17, hi=0.27)
    workload("kg_t17", 131072, 16, 0.008, 1.32, 18, 2048, 0.01)
    # Terabyte-shaped chunk (terabyte_like.cfg table 25, dim 64, 8192 rows)
    workload("tb_t25", 3072, 64, 0.0155, 0.36, 26, 8192, 0.03)
    with open(OUT, "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
