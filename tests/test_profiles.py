"""CPU: the controller's persistence and the bench workloads' fixtures.

* format_double / write_profiles / read_profiles (config.hpp:247-303,
  csv.hpp:31-37) are byte-identical to the reference's;
* the committed presets (configs/presets.json) and profile files
  (profiles_{kg,tb,sc}.cfg, written by the reference's offline_analysis via
  tests/golden/make_profiles.py) agree with workload.py's preset tables.
"""
import json
import os
import random
import struct

import pytest

from paper_2407_04272_b200 import policy as P
from paper_2407_04272_b200 import workload as W

GOLD = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "configs")


def test_format_double_matches_reference(ref):
    rng = random.Random(7)
    vals = [0.0, -0.0, 1.0, 3.0, 0.05, 0.01, 1e-300, 5e-324, 1e16, 1e15, 123456789012345680000.0, 1e21, 0.1 + 0.2,
            1.7976931348623157e308, 100.0, 1234.5, 1e-5, 1e-4, 0.001, 2.5e-7]
    vals += [struct.unpack("<d", struct.pack("<Q", rng.getrandbits(64)))[0] for _ in range(3000)]
    vals += [rng.uniform(0, 1) * 10 ** rng.randint(-30, 30) for _ in range(3000)]
    vals += [float(rng.randint(0, 10 ** rng.randint(1, 25))) for _ in range(1000)]
    for v in vals:
        if v != v or v in (float("inf"), float("-inf")):
            continue
        assert P.format_double(v) == ref.format_double(v), v


@pytest.mark.parametrize("wl", ["kg", "tb", "sc"])
def test_profiles_roundtrip_bytes(ref, tmp_path, wl):
    """read_profiles then write_profiles reproduces the reference's file byte
    for byte, and the reference reads our parse back identically."""
    src = os.path.join(GOLD, f"profiles_{wl}.cfg")
    prof = P.read_profiles(src)
    out = tmp_path / "p.cfg"
    P.write_profiles(str(out), prof)
    assert out.read_bytes() == open(src, "rb").read()
    back = ref.read_profiles(str(out))
    for t, p in prof.items():
        assert back[t]["codec"] == p.codec and back[t]["eb"] == p.eb and back[t]["cls"] == p.cls
        assert back[t]["n_original"] == p.n_original_patterns and back[t]["n_quantized"] == p.n_quantized_patterns


def test_read_profiles_errors(tmp_path):
    bad = tmp_path / "b.cfg"
    bad.write_text("profiles.count = 1\nprofile.0.table = 0\n")
    with pytest.raises(P._lib.CodecConfigError, match="missing config key 'profile.0.n_original'"):
        P.read_profiles(str(bad))
    bad.write_text("profiles.count = x\n")
    with pytest.raises(P._lib.CodecConfigError, match="expects a non-negative integer"):
        P.read_profiles(str(bad))
    bad.write_text("no equals sign\n")
    with pytest.raises(P._lib.CodecConfigError, match="expected 'key = value'"):
        P.read_profiles(str(bad))
    with pytest.raises(P._lib.CodecConfigError, match="cannot open config file"):
        P.read_profiles(str(tmp_path / "missing.cfg"))


def test_presets_match_workload_tables():
    with open(os.path.join(GOLD, "presets.json")) as f:
        g = json.load(f)
    assert [tuple(t) for t in g["presets"]["kaggle_like.cfg"]["tables"]] == \
        [tuple(float(x) for x in t) for t in W.KAGGLE_TABLES]
    assert [tuple(t) for t in g["presets"]["terabyte_like.cfg"]["tables"]] == \
        [tuple(float(x) for x in t) for t in W.TERABYTE_TABLES]
    for wl in ("kg", "tb", "sc"):
        w = g["workloads"][wl]
        prof = P.read_profiles(os.path.join(GOLD, w["profiles"]))
        assert sorted(prof) == list(range(w["tables"]))
        geb = w["global_eb"]
        for p in prof.values():
            assert p.eb in (geb * 5 / 3, geb, geb / 3) or abs(p.eb - geb * (5 / 3)) < 1e-15
            assert p.codec in (1, 2)
