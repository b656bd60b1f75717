"""GPU: the reference's Simulator with the GPU codec (embc_simulate) against the
reference Simulator itself (oracle/_ref, run_training_schedule) at 2..8 ranks:
per-iteration uncompressed / payload / metadata bytes, max abs error, the
delivered-value digest of every rank's decoded doubles, and
SimReport::deterministic_digest are identical (commsim_test.cc:57-101 style).
This is multi-rank parity of the GPU data path (compress -> pack -> metadata ->
unpack -> decode) on one device."""
import ctypes as C

import numpy as np
import pytest

from paper_2407_04272_b200 import policy as P
from paper_2407_04272_b200 import simulate as S
from paper_2407_04272_b200 import workload as W

pytestmark = pytest.mark.gpu


def _ref_sim(ref, cfg, profiles):
    n, T = cfg.iterations, len(cfg.tables)
    arr = {k: np.zeros(n, np.uint64) for k in ("unc", "pay", "meta", "dig")}
    maxerr = np.zeros(n, np.float64)
    cols = list(zip(*cfg.tables))
    rows = np.array(cols[0], np.uint32)
    dims = np.array(cols[1], np.uint32)
    dist = np.array(cols[2], np.int32)
    mu, sig, lo, hi, zf = (np.array(cols[k], np.float64) for k in range(3, 8))
    R = cfg.ranks
    pc = np.array([profiles[r].codec for r in range(R)], np.uint8)
    pe = np.array([profiles[r].eb for r in range(R)], np.float64)
    rep = C.c_uint64()
    err = C.create_string_buffer(512)
    p = lambda x: x.ctypes.data_as(C.c_void_p)  # noqa: E731
    d = cfg.policy.decay
    rc = ref.L.ref_simulate(R, cfg.batch, n, cfg.seed, int(cfg.compression), cfg.policy.global_eb, d.start_scale,
                            d.decay_end, d.step_count, p(rows), p(dims), p(dist), p(mu), p(sig), p(lo), p(hi), p(zf),
                            T, p(pc), p(pe), p(arr["unc"]), p(arr["pay"]), p(arr["meta"]), p(maxerr), p(arr["dig"]),
                            C.byref(rep), err, 512)
    assert rc == 0, err.value
    return arr, maxerr, rep.value


def _tables(preset, k, dim):
    out = []
    for t in range(k):
        rows, dist, mu, sigma, lo, hi, zipf = preset[t % len(preset)]
        out.append((rows, dim, dist, mu, sigma, lo, hi, zipf))
    return out


CASES = [
    # ranks, batch, iters, seed, tables (preset, count, dim), codecs per rank, ebs per rank, decay
    (2, 128, 4, 7, (W.KAGGLE_TABLES, 2, 8), [1, 2], [0.02, 0.01], ("stepwise", 2.0, 4, 3)),
    (4, 256, 5, 11, (W.TERABYTE_TABLES, 4, 16), [0, 1, 2, 1], [0.01, 0.03, 0.02, 0.05], ("stepwise", 2.0, 4, 4)),
    (8, 192, 3, 3, (W.KAGGLE_TABLES[5:], 3, 32), [2, 1, 2, 1, 0, 2, 1, 2], [0.01] * 8, ("stepwise", 1.0, 0, 4)),
    (3, 512, 2, 5, (W.TERABYTE_TABLES[10:], 5, 64), [1, 1, 2], [1e-3, 0.03, 0.01], ("stepwise", 2.0, 2, 2)),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_gpu_simulator_matches_reference(ref, case):
    R, B, iters, seed, (preset, k, dim), codecs, ebs, (fn, s0, end, steps) = CASES[case]
    cfg = S.SimConfig(ranks=R, batch=B, iterations=iters, seed=seed,
                      policy=P.PolicyConfig(global_eb=0.02, decay=P.DecayConfig(fn, s0, end, steps)),
                      tables=_tables(preset, k, dim))
    profiles = {r: P.TableProfile(r, codec=codecs[r], eb=ebs[r]) for r in range(R)}
    got = S.run_training_schedule(cfg, profiles)
    arr, maxerr, rep = _ref_sim(ref, cfg, profiles)
    for i, it in enumerate(got.iterations):
        assert it.uncompressed_bytes == arr["unc"][i], (case, i)
        assert it.payload_bytes == arr["pay"][i], (case, i)
        assert it.metadata_bytes == arr["meta"][i], (case, i)
        assert it.max_abs_error == maxerr[i], (case, i)
        assert it.delivered_digest == int(arr["dig"][i]), (case, i)
        assert it.comp_time > 0 and it.decomp_time > 0
    assert got.deterministic_digest == rep, case


def test_gpu_simulator_baseline_matches_reference(ref):
    """Compression off: raw fp32 delivery, payload = uncompressed, no metadata."""
    cfg = S.SimConfig(ranks=3, batch=100, iterations=2, seed=9, compression=False,
                      policy=P.PolicyConfig(global_eb=0.02), tables=_tables(W.KAGGLE_TABLES, 3, 8))
    profiles = {r: P.TableProfile(r, codec=1, eb=0.02) for r in range(3)}
    got = S.run_training_schedule(cfg, profiles)
    arr, maxerr, rep = _ref_sim(ref, cfg, profiles)
    for i, it in enumerate(got.iterations):
        assert (it.uncompressed_bytes, it.payload_bytes, it.metadata_bytes) == (arr["unc"][i], arr["pay"][i],
                                                                             arr["meta"][i])
        assert it.delivered_digest == int(arr["dig"][i])
        assert it.max_abs_error == 0.0
    assert got.deterministic_digest == rep
