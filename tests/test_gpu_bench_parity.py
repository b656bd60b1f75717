"""GPU parity on the exact configurations the bench measures, against the
reference itself (oracle/_ref: the unmodified headers).

* Kaggle-shaped step (BASELINE configs[1]): 26 x [2048, 16] with the
  reference's offline_analysis bounds and codecs (configs/profiles_kg.cfg), one
  packed call through the single-launch encoder -- bytes == the reference's
  pack(encode_chunks(jobs)), decoded values == the reference's decode_chunk.
* Terabyte-shaped slice (configs[2]): 26 x [8192, 64], one packed call through
  the two-pass encoder (k_stats / k_sizes / k_emit).
* Scaled-DLRM chunks (configs[4]): dim 128, 4 / 8 / 16 MiB chunks.
* A bound from eb_at in the middle of the stepwise decay (policy.hpp:336-342).
* offline_analysis on the GPU (pattern counts on the device, codec by Eq. 2 at
  B -> 0) == the reference's classes, bounds and codecs.
"""
import numpy as np
import pytest
import torch

from paper_2407_04272_b200 import _lib
from paper_2407_04272_b200 import codec as K
from paper_2407_04272_b200 import policy as P
from paper_2407_04272_b200 import workload as W

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def step_inputs(wl, it, R=1, dst=0, tables=None):
    specs = W.workload_specs(wl)
    w = W.WORKLOADS[wl]
    B = w["batch"](R)
    out = []
    for t in (tables if tables is not None else range(w["tables"])):
        tab = W.gen_table(specs[t])
        out.append(tab[W.lookup_indices(specs[t], B, W.lookup_stream(it, t, dst, R))])
    return out


def kernels_of(ctx, fn):
    ctx.timing(True)
    fn()
    names = [n for n, _ in ctx.timing_collect()]
    ctx.timing(False)
    return names


def check_packed_vs_reference(ctx, ref, xs, ebs, codecs, expect_kernels):
    jobs = [K.EncodeJob(torch.from_numpy(x).to(DEV), eb, c) for x, eb, c in zip(xs, ebs, codecs)]
    res = {}
    names = kernels_of(ctx, lambda: res.setdefault("r", K.encode_chunks(jobs, K.LAYOUT_PACKED)))
    for k in expect_kernels:
        assert k in names, (k, names)
    got = bytes(res["r"].buffer.cpu().numpy().tobytes())
    want = ref.encode_pack([x.astype(np.float64) for x in xs], ebs, codecs, workers=8)
    assert len(got) == len(want)
    assert got == want
    outs64 = K.decode_packed(got, K.OUT_F64)
    assert K.decode_fallbacks() == 0
    outs32 = K.decode_packed(got, K.OUT_F32)
    chunks = ref.unpack(want)
    for j, (c, o64, o32) in enumerate(zip(chunks, outs64, outs32)):
        d = ref.decode_chunk(c)
        assert np.array_equal(o64.cpu().numpy().view(np.uint64), d.view(np.uint64)), j
        assert np.array_equal(o32.cpu().numpy(), d.astype(np.float32)), j
        assert np.abs(d - xs[j].astype(np.float64)).max() <= ebs[j]
    return len(got)


@pytest.mark.parametrize("it", [0, 7])
def test_kaggle_step_bytes_equal_reference(ctx, ref, it):
    prof = W.workload_profiles("kg")
    xs = step_inputs("kg", it)
    T = len(xs)
    n = check_packed_vs_reference(ctx, ref, xs, [prof[t].eb for t in range(T)], [prof[t].codec for t in range(T)],
                                  ["k_encode"])
    assert 26 * 2048 * 16 * 4 / n > 10  # the step's compression ratio (both sides)


def test_terabyte_slice_two_pass_bytes_equal_reference(ctx, ref):
    prof = W.workload_profiles("tb")
    xs = step_inputs("tb", 3)
    T = len(xs)
    check_packed_vs_reference(ctx, ref, xs, [prof[t].eb for t in range(T)], [prof[t].codec for t in range(T)],
                              ["k_stats", "k_sizes", "k_emit"])


@pytest.mark.parametrize("R", [8, 4, 2])
def test_scaled_chunks_bytes_equal_reference(ctx, ref, R):
    """configs[4] chunks [65536/R, 128]: 4 / 8 / 16 MiB each."""
    prof = W.workload_profiles("sc")
    tables = [0, 7, 12, 33]  # vlz, huffman (eb 0.01 / 0.03 / 0.05 classes among them)
    xs = step_inputs("sc", 1, R=R, dst=R - 1, tables=tables)
    assert xs[0].shape == (65536 // R, 128)
    check_packed_vs_reference(ctx, ref, xs, [prof[t].eb for t in tables], [prof[t].codec for t in tables],
                              [])


def test_mid_decay_bound_bytes_equal_reference(ctx, ref):
    """eb_at with the stepwise decay 2 -> 1 over 500 iterations (configs[3]) at
    iteration 300: multiplier 4/3, a bound that is not a round number."""
    cfg = P.PolicyConfig(global_eb=0.03, decay=P.DecayConfig("stepwise", 2.0, 500, 4))
    for wl, tables in (("kg", [3, 9, 16]), ("tb", [0, 12, 23])):
        prof = W.workload_profiles(wl)
        ebs = [P.eb_at(t, 300, prof, cfg) for t in tables]
        assert all(e == prof[t].eb * ref.decay_multiplier(300, 0, 2.0, 500, 4) for e, t in zip(ebs, tables))
        assert ebs[0] != prof[tables[0]].eb
        xs = step_inputs(wl, 300, tables=tables)
        check_packed_vs_reference(ctx, ref, xs, ebs, [prof[t].codec for t in tables], [])


@pytest.mark.parametrize("wl", ["kg", "tb", "sc"])
def test_offline_analysis_matches_reference(ctx, wl):
    """offline_analysis (policy.hpp:278-302) of the iteration-0 samples on the
    GPU: pattern counts, survival, class, bound and codec equal the profiles the
    reference wrote (configs/profiles_<wl>.cfg, policy_test.cc:197-225 shape)."""
    want = W.workload_profiles(wl)
    specs = W.workload_specs(wl)
    B = 8192 if wl == "sc" else W.WORKLOADS[wl]["batch"](1)
    tables = range(W.WORKLOADS[wl]["tables"]) if wl != "sc" else range(0, 64, 3)
    samples = {t: W.Table(specs[t], DEV).lookup_batch(B, 0) for t in tables}
    cfg = P.PolicyConfig(global_eb=W.WORKLOADS[wl]["global_eb"])
    got = P.offline_analysis(samples, cfg, bandwidth=1e-300, timed=False)
    for t in tables:
        g, w = got[t], want[t]
        assert (g.n_original_patterns, g.n_quantized_patterns) == (w.n_original_patterns, w.n_quantized_patterns), t
        assert (g.survival_ratio, g.homo_index, g.cls, g.eb, g.codec) == \
            (w.survival_ratio, w.homo_index, w.cls, w.eb, w.codec), t
        ratios = {m.codec: m.ratio for m in g.measured}
        for m in w.measured:
            assert ratios[m.codec] == m.ratio, (t, m.codec)


def test_invalid_window_value_error(ctx, ref):
    """VlzConfig::validate (vlz.hpp:39-43): window outside [1, 65536] is a
    ValueError with the reference's text, from encode and from match_stats."""
    x = (np.arange(64, dtype=np.float32) % 5 * 0.02).reshape(16, 4)
    for w in (0, 65537, 1 << 20):
        with pytest.raises(Exception) as r:
            ref.encode_chunk(x.astype(np.float64), 4, 0.01, 1, w)
        with pytest.raises(_lib.CodecValueError) as g:
            K.encode_chunk(torch.from_numpy(x).to(DEV), 0.01, K.CODEC_VLZ, w)
        assert str(g.value) == r.value.msg
        with pytest.raises(_lib.CodecValueError) as g2:
            K.match_stats(K.quantize(torch.from_numpy(x).to(DEV), 0.01), w)
        assert str(g2.value) == r.value.msg
    # raw and huffman chunks ignore the window, as in the reference
    for c in (0, 2):
        assert K.encode_chunk(torch.from_numpy(x).to(DEV), 0.01, c, 0) == \
            ref.encode_chunk(x.astype(np.float64), 4, 0.01, c, 0)


def test_select_codec_timed_eq2(ctx):
    """select_codec (policy.hpp:239-274) with measured GPU throughputs
    (SURVEY 8(f) row 2): the ratios equal the untimed (pinned) run's, the
    throughputs are positive, the choice is the argmax of Eq. 2
    (estimate_speedup, policy.hpp:202-208) over the measured samples with ties
    to the lower codec tag, and at B -> 0 it reduces to the ratio choice the
    reference pinned.  B = the NVLink per-direction bandwidth."""
    wl = "kg"
    prof = W.workload_profiles(wl)
    specs = W.workload_specs(wl)
    B = W.WORKLOADS[wl]["batch"](1)
    cands = [K.CODEC_VLZ, K.CODEC_HUFFMAN]
    for t in (0, 7, 23):
        sample = W.Table(specs[t], DEV).lookup_batch(B, 0)
        pinned, pm = P.select_codec(sample, prof[t].eb, cands, 1e-300, timed=False)
        assert pinned == prof[t].codec
        for bw in (900e9, 1e-300):
            chosen, ms = P.select_codec(sample, prof[t].eb, cands, bw, timed=True)
            assert [m.ratio for m in ms] == [m.ratio for m in pm]
            assert all(m.comp_bps > 0 and m.decomp_bps > 0 and np.isfinite(m.comp_bps) for m in ms)
            sp = [P.estimate_speedup(m.ratio, bw, m.comp_bps, m.decomp_bps) for m in ms]
            best = max(range(len(ms)), key=lambda i: (sp[i], -ms[i].codec))
            want = ms[best].codec if ms[best].ratio > 1.0 else K.CODEC_RAW
            assert chosen == want, (t, bw, sp)
            if bw < 1.0:
                assert chosen == pinned


def test_pipelined_chain_graph_equals_eager(ctx):
    """The bench's pipelined schedule as a library user would run it: two codec
    contexts on two streams, several steps captured in one CUDA graph with no
    join between steps (compress of k+1 may overlap decode of k; decode of k
    waits for compress of k only).  Every step's packed bytes and decoded
    values equal the eager (serial) call's."""
    prof = W.workload_profiles("kg")
    T = 26
    ebs, codecs = [prof[t].eb for t in range(T)], [prof[t].codec for t in range(T)]
    S = 4
    sets = []
    for it in range(S):
        x = [torch.from_numpy(a).to(DEV) for a in step_inputs("kg", it)]
        jobs = [K.EncodeJob(x[t], ebs[t], codecs[t]) for t in range(T)]
        r = K.encode_chunks(jobs, K.LAYOUT_PACKED)
        want = bytes(r.buffer[: r.total].cpu().numpy().tobytes())
        table = K.unpack_table(want)
        y = [torch.empty_like(x[t]) for t in range(T)]
        refs = []
        for t, (o, ln) in enumerate(table):
            cr = _lib.ChunkRef()
            cr.offset, cr.length, cr.out, cr.dim, cr.count, cr.codec = o, ln, y[t].data_ptr(), 16, x[t].shape[0], codecs[t]
            refs.append(cr)
        out = torch.zeros(r.total + 256, dtype=torch.uint8, device=DEV)
        sets.append({"x": x, "cj": [j.to_c() for j in jobs], "want": want, "y": y, "refs": refs, "out": out})
    # eager decode of the reference bytes: the values every pipelined decode must reproduce
    expect = []
    for s in sets:
        s["out"][: len(s["want"])].copy_(torch.frombuffer(bytearray(s["want"]), dtype=torch.uint8).to(DEV))
        ctx.decode_raw(s["out"], s["refs"], K.OUT_F32, False)
        ctx.sync()
        expect.append([yy.clone() for yy in s["y"]])
    for s in sets:
        s["out"].zero_()
        for yy in s["y"]:
            yy.fill_(float("nan"))
    ectx, dctx = K.Context(0), K.Context(0)
    ectx.reserve_capture(64 << 20)
    dctx.reserve_capture(64 << 20)
    # size the decode context's scratch before capture (as the bench does)
    for s in sets:
        s["out"][: len(s["want"])].copy_(torch.frombuffer(bytearray(s["want"]), dtype=torch.uint8).to(DEV))
        dctx.decode_raw(s["out"], s["refs"], K.OUT_F32, False)
        ectx.encode_raw(s["cj"], K.LAYOUT_PACKED, s["out"])
    torch.cuda.synchronize()
    ectx.sync()
    dctx.sync()
    for s in sets:
        s["out"].zero_()
        for yy in s["y"]:
            yy.fill_(float("nan"))
    torch.cuda.synchronize()
    s_enc, s_dec, s_cap = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s_cap):
        s_enc.wait_stream(s_cap)
        s_dec.wait_stream(s_cap)
        for k in range(S + 1):  # compress k (k < S) beside decode k - 1 (k > 0)
            if k < S:
                ectx.encode_raw(sets[k]["cj"], K.LAYOUT_PACKED, sets[k]["out"], stream=s_enc)
            if k > 0:
                dctx.decode_raw(sets[k - 1]["out"], sets[k - 1]["refs"], K.OUT_F32, False, stream=s_dec)
            if k < S:
                ev = torch.cuda.Event()
                ev.record(s_enc)
                s_dec.wait_event(ev)
        s_cap.wait_stream(s_enc)
        s_cap.wait_stream(s_dec)
    g.replay()
    torch.cuda.synchronize()
    for k, s in enumerate(sets):
        assert bytes(s["out"][: len(s["want"])].cpu().numpy().tobytes()) == s["want"], k
        for t in range(T):
            assert torch.equal(s["y"][t], expect[k][t]), (k, t)
            assert (s["y"][t].double() - s["x"][t].double()).abs().max().item() <= ebs[t]
