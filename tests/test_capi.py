"""CPU: the C-ABI library loads and exports every entry point include/embc_cuda.h
declares; host-side functions (controller arithmetic, workload generator) match
the reference.  No device compute here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2407_04272_b200 import _lib
from paper_2407_04272_b200 import workload as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "embc_cuda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(embc_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_header():
    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTS)
    assert L.embc_version().decode().endswith("sm_100a")


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_decay_and_classify_match_reference(ref):
    L = _lib.lib()
    v = C.c_double()
    for it in range(0, 1100, 13):
        for fn in (0, 1, 2):
            assert L.embc_decay_multiplier(it, fn, 2.0, 1000, 4, C.byref(v)) == 0
            assert v.value == ref.decay_multiplier(it, fn, 2.0, 1000, 4)
    assert L.embc_decay_multiplier(5, 0, 0.5, 10, 4, C.byref(v)) == _lib.ERR_CONFIG
    cls, eb = C.c_int(), C.c_double()
    for s in np.linspace(0.0, 1.0, 57):
        assert L.embc_classify_table(float(s), 0.03, 5 / 3, 3.0, 0.7, 0.95, C.byref(cls), C.byref(eb)) == 0
        rc, reb = ref.classify(float(s), 0.03, 5 / 3, 3.0, 0.7, 0.95)
        assert (cls.value, eb.value) == (rc, reb)
    assert L.embc_classify_table(0.5, 0.03, 5 / 3, 3.0, 0.95, 0.7, C.byref(cls), C.byref(eb)) == _lib.ERR_CONFIG
    for r in (1.0, 3.3, 19.9):
        assert L.embc_estimate_speedup(r, 4e9, 1e9, 2e9, C.byref(v)) == 0
        assert v.value == ref.estimate_speedup(r, 4e9, 1e9, 2e9)


def test_workload_generator_matches_reference(ref):
    for t, (rows, dist, mu, sigma, lo, hi, zipf) in enumerate(W.TERABYTE_TABLES[:8]):
        spec = W.TableSpec(rows, 16, dist, mu, sigma, lo, hi, zipf, W.table_seed(1, t), t)
        a = W.gen_table(spec)
        b = ref.gen_table(rows, 16, dist, mu, sigma, lo, hi, zipf, spec.seed)
        assert np.array_equal(a.astype(np.float64), b)
        ia = W.lookup_indices(spec, 500, stream=3 + t)
        ib = ref.lookup_indices(rows, 16, zipf, spec.seed, 500, 3 + t, dist, mu, sigma, lo, hi)
        assert np.array_equal(ia, ib)
    assert W.mix_seed(1, 0x7AB1E) == ref.mix_seed(1, 0x7AB1E)


def test_workload_golden_inputs(golden):
    import hashlib
    for w in golden["workloads"]:
        spec = W.TableSpec(w["rows"], w["dim"], w["dist"], 0.0, w["sigma"], w["lo"], w["hi"], w["zipf"], w["seed"])
        x = W.gen_table(spec)[W.lookup_indices(spec, w["batch"], w["stream"])]
        assert hashlib.sha256(x.tobytes()).hexdigest() == w["x_sha"], w["name"]


def test_unpack_matches_reference(ref):
    """embc_unpack (host, no device work) == the reference's unpack()
    (container.hpp:258-292): offsets/lengths, and the FormatError text for
    gaps, overlaps, overruns, trailing bytes and truncated tables."""
    from oracle import OracleError
    from paper_2407_04272_b200 import codec as K
    rng = np.random.default_rng(5)
    x = (rng.standard_normal(64) * 0.1)
    chunks = [ref.encode_chunk(x[:8 * k], 8, 0.01, k % 3) for k in range(1, 5)]
    good = ref.pack(chunks)
    table = K.unpack_table(good)
    assert [good[o:o + n] for o, n in table] == chunks
    assert K.unpack_table(ref.pack([])) == []
    cases = [good[:3], good[:11], good + b"\0", good[:-1], bytearray(good), bytearray(good), bytearray(good)]
    cases[4][4] ^= 1                      # first offset skips a byte
    cases[5][12:20] = (1 << 40).to_bytes(8, "little")  # length runs past the end
    cases[6][0] = 200                     # rank count larger than the table
    for buf in cases:
        buf = bytes(buf)
        with pytest.raises(OracleError) as r:
            ref.unpack(buf)
        with pytest.raises(_lib.CodecFormatError) as g:
            K.unpack_table(buf)
        assert str(g.value) == r.value.msg, buf[:24].hex()
