"""GPU parity: the sm_100a codec (through the C ABI) against the oracle
restatement, the reference itself (oracle/_ref) and the golden fixtures.

Bar: bit-exact bytes for every chunk/stream; decoded values bit-exact in fp64
mode and equal to float(reference double) in fp32 mode; failures raise the
reference's exception class (and message, where oracle/_ref is present)."""
import hashlib

import numpy as np
import pytest
import torch

from oracle import OracleError
from paper_2407_04272_b200 import _lib
from paper_2407_04272_b200 import codec as K
from paper_2407_04272_b200 import workload as W

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def sha(b):
    return hashlib.sha256(b).hexdigest()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def gpu_encode(x32: np.ndarray, dim, eb, codec, window=255):
    return K.encode_chunk(dev(x32.reshape(-1, dim)), eb, codec, window)


# ---------------------------------------------------------------- quantizer

def test_quantize_literal_goldens(ctx, golden):
    for q in golden["literal"]["quantize"]:
        got = K.quantize(dev(np.array(q["values"], np.float64)), q["eb"])
        assert got.cpu().tolist() == q["codes"]


def test_quantize_fp32_fuzz_and_bin_edges(ctx, oracle):
    rng = np.random.default_rng(11)
    for trial in range(60):
        eb = float(10 ** rng.uniform(-5, 0))
        x = (rng.standard_normal(20000) * 10 ** rng.uniform(-3, 1)).astype(np.float32)
        # fp32-rounded bin edges (k + 1/2) * 2eb and their neighbours
        k = rng.integers(-3000, 3000, 4000)
        edges = ((k + 0.5) * 2 * eb).astype(np.float32)
        x = np.concatenate([x, edges, np.nextafter(edges, np.float32(np.inf)),
                            np.nextafter(edges, np.float32(-np.inf)), np.float32([0.0, -0.0])])
        try:
            want = oracle.quantize(x, eb)
        except OracleError as e:
            with pytest.raises(_lib.CodecValueError) as ge:
                K.quantize(dev(x), eb)
            assert ge.value.index == e.index
            continue
        got = K.quantize(dev(x), eb).cpu().numpy()
        assert np.array_equal(got, want), trial


def test_quantize_errors_first_index(ctx, ref):
    x = np.zeros(5000, np.float32)
    x[3777] = np.nan
    x[4000] = np.inf
    with pytest.raises(_lib.CodecValueError) as e:
        K.quantize(dev(x), 0.01)
    assert str(e.value) == "non-finite value at index 3777"
    with pytest.raises(_lib.CodecValueError) as e:
        K.quantize(dev(np.array([0.0, 3.0e9], np.float32)), 1e-4)
    with pytest.raises(OracleError) as r:
        ref.quantize(np.array([0.0, 3.0e9]), 1e-4)
    assert str(e.value) == r.value.msg


def test_dequantize_bits(ctx, oracle):
    rng = np.random.default_rng(5)
    codes = rng.integers(-(2 ** 31) + 1, 2 ** 31 - 1, 100000).astype(np.int32)
    for eb in (1e-3, 0.017, 3.3e-7):
        want = oracle.dequantize(codes, eb)
        got = K.dequantize(dev(codes), eb, torch.float64).cpu().numpy()
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
        got32 = K.dequantize(dev(codes), eb, torch.float32).cpu().numpy()
        assert np.array_equal(got32, want.astype(np.float32))


# ---------------------------------------------------------------- chunks

def test_literal_chunk_and_streams(ctx, golden):
    L = golden["literal"]
    c = L["chunk_raw"]
    assert gpu_encode(np.array(c["values"], np.float32), 2, c["eb"], 0).hex() == c["bytes"]
    for v in L["vlz"]:
        toks = K.vlz_encode(dev(np.array(v["codes"], np.int32).reshape(-1, v["dim"])), v["window"])
        assert toks.hex() == v["tokens"]
        back = K.vlz_decode(bytes.fromhex(v["tokens"]), v["dim"], len(v["codes"]) // v["dim"])
        assert back.cpu().numpy().ravel().tolist() == v["codes"]
    assert K.match_stats(dev(np.array(L["vlz"][0]["codes"], np.int32).reshape(-1, 2)), 32) == (1, 3)
    w = L["vlz_window"]
    assert K.match_stats(dev(np.array(w["codes"], np.int32).reshape(-1, 1)), 2)[1] == w["refs_w2"]
    assert K.match_stats(dev(np.array(w["codes"], np.int32).reshape(-1, 1)), 3)[1] == w["refs_w3"]
    h = L["huff_textbook"]
    assert K.huff_encode(dev(np.array(h["codes"], np.int32))).hex() == h["stream"]
    h = L["huff_1000"]
    s = K.huff_encode(dev(np.full(h["count"], h["symbol"], np.int32)))
    assert s.hex() == h["stream"]
    assert K.huff_decode(s, h["count"]).cpu().tolist() == [h["symbol"]] * h["count"]


def test_workload_digests(ctx, golden):
    """BASELINE-shaped seeded workloads: GPU bytes/values == reference digests."""
    for w in golden["workloads"]:
        spec = W.TableSpec(w["rows"], w["dim"], w["dist"], 0.0, w["sigma"], w["lo"], w["hi"], w["zipf"], w["seed"])
        x = W.gen_table(spec)[W.lookup_indices(spec, w["batch"], w["stream"])]
        assert sha(x.tobytes()) == w["x_sha"]
        xd = dev(x)
        for key, c in w["chunks"].items():
            codec, win = map(int, key.split(":"))
            b = K.encode_chunk(xd, w["eb"], codec, win)
            assert len(b) == c["len"] and sha(b) == c["sha"], (w["name"], key)
            d64 = K.decode_chunk(b, K.OUT_F64).cpu().numpy()
            assert K.decode_fallbacks() == 0, (w["name"], key)  # parallel decoders handled it
            assert sha(d64.tobytes()) == c["dec_sha"], (w["name"], key)
            d32 = K.decode_chunk(b, K.OUT_F32).cpu().numpy()
            assert sha(d32.tobytes()) == c["dec32_sha"], (w["name"], key)
            assert np.abs(d64 - x.astype(np.float64)).max() <= w["eb"]  # error bound, in f64
        codes = K.quantize(xd, w["eb"])
        assert list(K.match_stats(codes, 255)) == w["match_stats"]
        assert list(K.pattern_counts(xd, w["eb"])) == w["pattern_counts"]


def _fuzz_batch(rng, trial):
    dim = int(rng.choice([1, 2, 3, 5, 8, 16, 17, 33, 64, 128]))
    n = int(rng.integers(0, 700))
    kind = trial % 4
    if kind == 0:
        x = rng.standard_normal(dim * n) * 0.1
    elif kind == 1:  # narrow alphabet -> repeated rows
        x = rng.integers(-3, 4, dim * n) * 0.02
    elif kind == 2:  # few distinct rows (Zipf-like lookups)
        rows = rng.standard_normal((int(rng.integers(1, 20)), dim)) * 0.05
        x = rows[rng.integers(0, len(rows), n)].ravel() if n else np.zeros(0)
    else:
        x = rng.random(dim * n) * 2 - 1
    return x.astype(np.float32), dim, n


def test_encode_decode_fuzz_vs_oracle(ctx, oracle):
    rng = np.random.default_rng(2027)
    for trial in range(240):
        x, dim, n = _fuzz_batch(rng, trial)
        eb = float(10 ** rng.uniform(-4, -1))
        codec = int(rng.integers(0, 3))
        win = int(rng.choice([1, 2, 7, 32, 255, 1024, 65536]))
        try:
            want = oracle.encode_chunk(x.astype(np.float64), dim, eb, codec, win)
        except OracleError as e:
            with pytest.raises(_lib.EmbcError) as ge:
                gpu_encode(x, dim, eb, codec, win)
            assert ge.value.status == (_lib.ERR_VALUE if e.kind == "value" else _lib.ERR_FORMAT)
            continue
        got = gpu_encode(x, dim, eb, codec, win)
        assert got == want, (trial, dim, n, codec, win)
        d = K.decode_chunk(got, K.OUT_F64).cpu().numpy().ravel()
        assert np.array_equal(d.view(np.uint64), oracle.decode_chunk(want).ravel().view(np.uint64)), trial


def test_acceptance_soundness_1e6(ctx):
    """acceptance_test.cc:103-141: >= 1e6 values, every codec, point-wise |x - x'| <= eb (in f64)."""
    rng = np.random.default_rng(0xACCE97)
    checked = 0
    rnd = 0
    while checked < 1_000_000:
        dim = int(rng.integers(1, 17))
        count = int(rng.integers(256, 768))
        if rnd % 2 == 0:
            x = (0.1 * rng.standard_normal(dim * count)).astype(np.float32)
        else:
            x = (rng.random(dim * count) * 2 - 1).astype(np.float32)
        eb = float(10 ** (-4 + 3 * rng.random()))
        b = gpu_encode(x, dim, eb, rnd % 3)
        d = K.decode_chunk(b, K.OUT_F64).cpu().numpy().ravel()
        assert np.abs(d - x.astype(np.float64)).max() <= eb
        checked += x.size
        rnd += 1


def test_vlz_codes_fuzz_vs_reference(ctx, ref):
    """vlz_test.cc:81-92 (2000-case round trip) + byte parity with the reference."""
    rng = np.random.default_rng(2026)
    windows = [1, 2, 7, 32, 255, 65536]
    for trial in range(400):
        dim = 1 + int(rng.integers(0, 6))
        n = int(rng.integers(0, 41))
        codes = (rng.integers(0, 5, dim * n) - 2).astype(np.int32)
        w = windows[trial % 6]
        toks = K.vlz_encode(dev(codes.reshape(-1, dim)), w)
        assert toks == ref.vlz_encode(codes, dim, w), trial
        back = K.vlz_decode(toks, dim, n).cpu().numpy().ravel()
        assert np.array_equal(back, codes)
        assert K.match_stats(dev(codes.reshape(-1, dim)), w) == ref.match_stats(codes, dim, w)


def test_huffman_codes_fuzz_vs_reference(ctx, ref):
    """huffman_test.cc:103-115 round trips + byte parity."""
    rng = np.random.default_rng(31)
    for trial in range(300):
        n = 1 + int(rng.integers(0, 400))
        alphabet = 1 + int(rng.integers(0, 64))
        codes = (rng.integers(0, alphabet, n) - alphabet // 2).astype(np.int32)
        s = K.huff_encode(dev(codes))
        assert s == ref.huff_encode(codes), trial
        assert np.array_equal(K.huff_decode(s, n).cpu().numpy(), codes)


def test_huffman_length_cap_and_empty(ctx, ref):
    # Fibonacci weights push the deepest leaf past 32 bits (huffman_test.cc:173-185)
    counts, a, b = [], 1, 1
    for _ in range(40):
        counts.append(a)
        a, b = b, a + b
    codes = np.repeat(np.arange(40, dtype=np.int32), counts[:40]) if sum(counts) < 50_000_000 else None
    sub = np.repeat(np.arange(34, dtype=np.int32), counts[:34])  # 34 Fibonacci symbols: depth 33
    with pytest.raises(_lib.CodecValueError) as e:
        K.huff_encode(dev(sub))
    with pytest.raises(OracleError) as r:
        ref.huff_encode(sub)
    assert str(e.value) == r.value.msg
    with pytest.raises(_lib.CodecValueError) as e:
        K.encode_chunk(torch.zeros((0, 4), dtype=torch.float32, device=DEV), 0.01, K.CODEC_HUFFMAN)
    assert str(e.value) == "huffman encoder requires a nonempty sequence"
    del codes


def test_malformed_streams_match_reference(ctx, ref):
    rng = np.random.default_rng(7)
    for trial in range(240):
        dim = int(rng.integers(1, 6))
        n = int(rng.integers(1, 40))
        codes = rng.integers(-2, 3, dim * n).astype(np.int32)
        is_vlz = trial % 2 == 1
        s = bytearray(ref.vlz_encode(codes, dim, 255) if is_vlz else ref.huff_encode(codes))
        k = int(rng.integers(0, 3))
        if k == 0 and len(s):
            del s[int(rng.integers(0, len(s))):]
        elif k == 1 and len(s):
            s[int(rng.integers(0, len(s)))] ^= int(rng.integers(1, 256))
        else:
            s += bytes([int(rng.integers(0, 256))])
        s = bytes(s)
        try:
            want = ("ok", (ref.vlz_decode(s, dim, n) if is_vlz else ref.huff_decode(s)).tobytes())
        except OracleError as e:
            want = ("err", e.kind, e.msg)
        try:
            if is_vlz:
                got = ("ok", K.vlz_decode(s, dim, n).cpu().numpy().tobytes())
            else:
                cnt = int.from_bytes(s[:8], "big") if len(s) >= 8 else 0
                if want[0] == "ok":
                    cnt = len(want[1]) // 4
                got = ("ok", K.huff_decode(s, cnt if cnt < 10_000_000 else 0).cpu().numpy().tobytes())
        except _lib.EmbcError as e:
            got = ("err", "value" if e.status == _lib.ERR_VALUE else "format", str(e))
        if want[:2] == ("err", "std"):
            assert got[0] == "err", trial
        elif want[0] == "err" and not is_vlz and "decoded" in got[-1]:
            assert got[0] == "err"
        else:
            assert got == want, (trial, is_vlz)


def test_chunk_container_errors(ctx, ref):
    good = gpu_encode(np.float32([0.01, -0.02, 0.03, 0.0]), 2, 0.01, 1)
    cases = []
    b = bytearray(good); b[0] = ord("X"); cases.append(bytes(b))
    b = bytearray(good); b[4] = 9; cases.append(bytes(b))
    b = bytearray(good); b[5] = 7; cases.append(bytes(b))
    cases.append(good + b"\x00")
    cases.append(good[:17])
    b = bytearray(good); b[6:14] = np.float64(-1.0).tobytes(); cases.append(bytes(b))
    raw = bytearray(gpu_encode(np.float32([0.01, -0.02]), 2, 0.01, 0))
    raw[18:22] = (3).to_bytes(4, "little")  # count 3 -> raw size mismatch
    cases.append(bytes(raw))
    for c in cases:
        with pytest.raises(OracleError) as r:
            ref.decode_chunk(c)
        with pytest.raises(_lib.EmbcError) as g:
            K.decode_chunk(c, K.OUT_F64)
        assert str(g.value) == r.value.msg
        assert (g.value.status == _lib.ERR_VALUE) == (r.value.kind == "value")


def test_pack_and_metadata_vs_reference(ctx, ref):
    rng = np.random.default_rng(18)
    for trial in range(30):
        jobs, ref_chunks = [], []
        for _ in range(int(rng.integers(0, 9))):
            x, dim, n = _fuzz_batch(rng, trial)
            if n == 0:
                x, n = np.zeros(dim, np.float32), 1
            codec = int(rng.integers(0, 3))
            jobs.append(K.EncodeJob(dev(x.reshape(n, dim)), 0.01, codec))
            ref_chunks.append(ref.encode_chunk(x.astype(np.float64), dim, 0.01, codec))
        packed = K.pack_encode(jobs)
        assert packed == ref.pack(ref_chunks), trial
        if jobs:
            r = K.encode_chunks(jobs, K.LAYOUT_CHUNKS, meta=True)
            meta = r.meta.cpu().numpy()
            for j, c in enumerate(ref_chunks):
                assert meta[j].tobytes() == ref.metadata(c)
        outs = K.decode_packed(packed, K.OUT_F64)
        for o, c in zip(outs, ref_chunks):
            assert np.array_equal(o.cpu().numpy().view(np.uint64), ref.decode_chunk(c).view(np.uint64))


def test_determinism_and_parallel_encode(ctx):
    """container_test.cc:241-255 / acceptance #10: identical bytes every run."""
    rng = np.random.default_rng(21)
    jobs = []
    for i in range(16):
        x = (rng.integers(-4, 5, 32 * 8) * 0.01).astype(np.float32)
        jobs.append(K.EncodeJob(dev(x.reshape(32, 8)), 0.01, i % 3))
    a = K.pack_encode(jobs)
    for _ in range(3):
        assert K.pack_encode(jobs) == a
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        b = K.pack_encode(jobs)
    assert a == b


def test_large_tb_chunk_roundtrip(ctx, ref):
    """Terabyte-shaped rank slice (8 tables x 8192 x 64, one packed call through
    the two-pass encoder): bytes == the reference's pack(encode_chunks(jobs)),
    deterministic, decoded bits == the reference's decode_chunk, within eb."""
    tables = W.preset_tables(W.TERABYTE_TABLES, 8, 64)
    jobs, xs = [], []
    for t, spec in enumerate(tables):
        x = W.gen_table(spec)[W.lookup_indices(spec, 8192, W.lookup_stream(0, t, 1, 8))]
        xs.append(x.astype(np.float64))
        jobs.append(K.EncodeJob(dev(x), 0.03, 1 + t % 2))
    r1 = K.encode_chunks(jobs, K.LAYOUT_PACKED)
    r2 = K.encode_chunks(jobs, K.LAYOUT_PACKED)
    assert torch.equal(r1.buffer, r2.buffer)
    got = bytes(r1.buffer.cpu().numpy().tobytes())
    want = ref.encode_pack(xs, [0.03] * 8, [1 + t % 2 for t in range(8)], workers=8)
    assert got == want
    outs = K.decode_packed(got, K.OUT_F64)
    assert K.decode_fallbacks() == 0
    for x, o, c in zip(xs, outs, ref.unpack(want)):
        d = o.cpu().numpy()
        assert np.array_equal(d.view(np.uint64), ref.decode_chunk(c).view(np.uint64))
        assert np.abs(d - x).max() <= 0.03


def test_long_huffman_codes_parallel_path(ctx, oracle):
    """Terabyte tables whose Huffman codes exceed the 11-bit prefix LUT (max
    length 16-17) decode on the parallel path, bit-exactly."""
    for t, eb in ((12, 0.01), (23, 0.01), (7, 0.01)):
        spec = W.TableSpec.preset(W.TERABYTE_TABLES, t, 64)
        x = W.gen_table(spec)[W.lookup_indices(spec, 8192, W.lookup_stream(0, t, 0, 1))]
        b = K.encode_chunk(dev(x), eb, K.CODEC_HUFFMAN)
        assert b == oracle.encode_chunk(x.astype(np.float64), 64, eb, 2)
        d = K.decode_chunk(b, K.OUT_F64).cpu().numpy()
        assert K.decode_fallbacks() == 0, t
        assert np.array_equal(d.view(np.uint64), oracle.decode_chunk(b).view(np.uint64))
