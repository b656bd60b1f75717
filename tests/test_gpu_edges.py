"""GPU parity on the envelope edges of the tiled kernels: rows wider than a
tile (single-row tiles, sequential VLZ decode past dim 1023), VLZ windows wider
than the staged hash window, Huffman alphabets past the one-warp codebook path
(block builder, global sort scratch, wide histogram pool) and past the 16-bit
symbol staging of the decoder, and a packed multi-chunk call mixing every
codec and shape.  Reference: the oracle restatement (pinned to the reference
by tests/test_oracle.py)."""
import numpy as np
import pytest
import torch

from paper_2407_04272_b200 import _lib
from paper_2407_04272_b200 import codec as K

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def roundtrip(oracle, x32, dim, eb, codec, window=255):
    want = oracle.encode_chunk(x32.astype(np.float64), dim, eb, codec, window)
    got = K.encode_chunk(dev(x32.reshape(-1, dim)), eb, codec, window)
    assert got == want, (dim, codec, window, len(got), len(want))
    d = K.decode_chunk(got, K.OUT_F64).cpu().numpy().ravel()
    assert np.array_equal(d.view(np.uint64), oracle.decode_chunk(want).ravel().view(np.uint64))
    f = K.decode_chunk(got, K.OUT_F32).cpu().numpy().ravel()
    assert np.array_equal(f, oracle.decode_chunk(want).ravel().astype(np.float32))
    return got


@pytest.mark.parametrize("dim", [1024, 2048, 4095, 4096, 5000, 8192])
def test_wide_rows(ctx, oracle, dim):
    rng = np.random.default_rng(dim)
    base = (rng.standard_normal((5, dim)) * 0.05).astype(np.float32)
    x = base[rng.integers(0, 5, 12)]  # repeated rows -> vlz references across single-row tiles
    for codec in (0, 1, 2):
        roundtrip(oracle, x.ravel(), dim, 0.01, codec)


def test_windows_past_the_hash_stage(ctx, oracle):
    rng = np.random.default_rng(5)
    rows = (rng.integers(-2, 3, (40, 2)) * 0.02).astype(np.float32)
    x = rows[rng.integers(0, 40, 6000)]
    for w in (1, 300, 2047, 2048, 4095, 65536):
        roundtrip(oracle, x.ravel(), 2, 0.01, 1, w)


def test_large_alphabets(ctx, oracle):
    rng = np.random.default_rng(9)
    # ~1500 symbols: block codebook builder, shared-memory sort
    x = (rng.standard_normal(60000) * 0.3).astype(np.float32)
    roundtrip(oracle, x, 4, 1e-3, 2)
    # > 4096-code span: wide histogram pool; > 1024 symbols sorted in global scratch
    x = (rng.standard_normal(80000) * 1.0).astype(np.float32)
    roundtrip(oracle, x, 8, 1e-4, 2)


def test_decoder_symbols_past_16_bits(ctx, oracle):
    # 70000 distinct codes: the decoder stores symbols straight to the output
    x = (np.arange(70000, dtype=np.float64) * 0.02 - 700.0).astype(np.float32)
    np.random.default_rng(3).shuffle(x)
    roundtrip(oracle, x, 7, 0.01, 2)


def test_packed_mixed_call(ctx, oracle):
    rng = np.random.default_rng(17)
    jobs, want = [], []
    shapes = [(2048, 16), (300, 64), (1, 3), (0, 8), (4096, 1), (64, 1500), (1000, 33)]
    for k, (n, dim) in enumerate(shapes):
        for codec in (0, 1, 2):
            if n == 0 and codec == 2:
                continue  # huffman on an empty batch is a ValueError (tested elsewhere)
            rows = (rng.standard_normal((max(1, n // 7), dim)) * 0.05).astype(np.float32)
            x = rows[rng.integers(0, len(rows), n)] if n else np.zeros((0, dim), np.float32)
            eb = [0.01, 0.003, 0.05][k % 3]
            jobs.append(K.EncodeJob(dev(x), eb, codec))
            want.append(oracle.encode_chunk(x.astype(np.float64).ravel(), dim, eb, codec))
    buf = K.pack_encode(jobs)
    table = K.unpack_table(buf)
    assert [buf[o:o + ln] for o, ln in table] == want
    outs = K.decode_packed(buf, K.OUT_F64)
    for o, w in zip(outs, want):
        assert np.array_equal(o.cpu().numpy().ravel().view(np.uint64), oracle.decode_chunk(w).ravel().view(np.uint64))
    # only the vlz chunk wider than the parallel decoder's envelope (dim > 1023) takes the sequential walker
    assert K.decode_fallbacks() == 1


def test_corrupted_long_streams_match_reference(ctx, ref):
    """Multi-segment vlz and multi-block huffman streams with a flipped,
    inserted or truncated byte: the parallel decoders either decode exactly
    what the reference decodes or raise the reference's error (via the exact
    sequential walkers)."""
    from oracle import OracleError
    from paper_2407_04272_b200 import _lib
    rng = np.random.default_rng(1234)
    for trial in range(150):
        is_vlz = trial % 2 == 0
        dim = int(rng.choice([3, 16, 64]))
        n = int(rng.integers(800, 3000))
        pool = rng.integers(-40, 41, (int(rng.integers(5, 200)), dim)).astype(np.int32)
        codes = pool[rng.integers(0, len(pool), n)].ravel()
        s = bytearray(ref.vlz_encode(codes, dim, 255) if is_vlz else ref.huff_encode(codes))
        k = trial % 3
        at = int(rng.integers(len(s) // 4, len(s)))
        if k == 0:
            s[at] ^= int(rng.integers(1, 256))
        elif k == 1:
            s.insert(at, int(rng.integers(0, 256)))
        else:
            del s[at:]
        s = bytes(s)
        try:
            want = ("ok", (ref.vlz_decode(s, dim, n) if is_vlz else ref.huff_decode(s)).tobytes())
        except OracleError as e:
            want = ("err", e.kind, e.msg)
        try:
            if is_vlz:
                got = ("ok", K.vlz_decode(s, dim, n).cpu().numpy().tobytes())
            else:
                got = ("ok", K.huff_decode(s, n * dim).cpu().numpy().tobytes())
        except _lib.EmbcError as e:
            got = ("err", "value" if e.status == _lib.ERR_VALUE else "format", str(e))
        if want[:2] == ("err", "std"):
            assert got[0] == "err", trial
        elif want[0] == "err" and not is_vlz and "decoded" in got[-1]:
            assert got[0] == "err", trial
        else:
            assert got == want, (trial, is_vlz, k)


@pytest.mark.parametrize("codec", [0, 1, 2])
def test_bin_edge_values_take_the_exact_path(ctx, oracle, codec):
    """Values at fp32-rounded bin edges ((k + 1/2) * 2eb) and large quotients
    fail the fast quantizer; the tile is redone on the exact binary64 path."""
    rng = np.random.default_rng(77 + codec)
    eb = 0.01
    k = rng.integers(-50, 50, 4096)
    x = ((k + 0.5) * (2 * eb)).astype(np.float32)
    x[::7] = (rng.standard_normal(len(x[::7])) * 0.1).astype(np.float32)
    x[5] = np.float32(30.0)  # |x / w| > 1024: exact path as well
    roundtrip(oracle, x, 16, eb, codec)


def test_two_pass_encode_large_call(ctx, oracle):
    """> 1024 tiles: the encoder runs its two-pass mode (sizes + layout, then
    bytes) instead of the fused single pass; bytes equal the reference's."""
    rng = np.random.default_rng(2048)
    jobs, want = [], []
    for t in range(5):
        pool = (rng.standard_normal((300, 128)) * 0.05).astype(np.float32)
        x = pool[rng.integers(0, 300, 8192)]
        codec = [1, 2, 0, 1, 2][t]
        jobs.append(K.EncodeJob(dev(x), 0.01, codec))
        want.append(oracle.encode_chunk(x.astype(np.float64).ravel(), 128, 0.01, codec))
    buf = K.pack_encode(jobs)
    table = K.unpack_table(buf)
    assert [buf[o:o + ln] for o, ln in table] == want


def test_two_pass_huffman_tile_spans(ctx, oracle):
    """Two-pass calls price a huffman tile from its E1 histogram when the
    tile's code span fits the kept window, else re-read it: a call of narrow
    tiles followed by one of wide tiles (spans > 256 codes) on the same
    context must not price the second from the first's histograms."""
    rng = np.random.default_rng(4096)
    for sigma in (0.02, 0.6, 0.02):
        jobs, want = [], []
        for t in range(3):
            x = (rng.standard_normal((12000, 128)) * sigma).astype(np.float32)
            jobs.append(K.EncodeJob(dev(x), 1e-3, 2))
            want.append(oracle.encode_chunk(x.astype(np.float64).ravel(), 128, 1e-3, 2))
        buf = K.pack_encode(jobs)
        table = K.unpack_table(buf)
        assert [buf[o:o + ln] for o, ln in table] == want, sigma


@pytest.mark.parametrize("dim,n,classes", [(16, 8192, 1), (64, 8192, 3), (4, 30000, 2), (1, 20000, 5)])
def test_long_reference_chains(ctx, oracle, dim, n, classes):
    # every row a repeat of a handful of rows: reference chains thousands of
    # rows deep, resolved by the copy tiles' pointer jumping
    rng = np.random.default_rng(dim * 7 + classes)
    rows = (rng.standard_normal((classes, dim)) * 0.05).astype(np.float32)
    x = rows[rng.integers(0, classes, n)]
    roundtrip(oracle, x.ravel(), dim, 0.01, 1)


def test_single_launch_encode_failure_then_recovery(ctx, oracle):
    """A quantization failure in one job of a Kaggle-shaped call (the
    single-launch encoder, every tile resident) reports the first failing
    job and value like encode_chunks, and the next call on the same context
    is byte-exact again (no state left behind by the aborted launch)."""
    rng = np.random.default_rng(26)
    xs = [(rng.standard_normal((2048, 16)) * 0.05).astype(np.float32) for _ in range(26)]
    codecs = [t % 3 for t in range(26)]
    bad = [x.copy() for x in xs]
    bad[17][5, 3] = np.nan
    bad[21][0, 0] = np.inf
    with pytest.raises(_lib.CodecValueError) as e:
        K.pack_encode([K.EncodeJob(dev(x), 0.01, c) for x, c in zip(bad, codecs)])
    assert e.value.job == 17 and e.value.index == 5 * 16 + 3
    assert str(e.value) == "non-finite value at index 83"
    want = [oracle.encode_chunk(x.astype(np.float64).ravel(), 16, 0.01, c) for x, c in zip(xs, codecs)]
    buf = K.pack_encode([K.EncodeJob(dev(x), 0.01, c) for x, c in zip(xs, codecs)])
    assert [buf[o:o + ln] for o, ln in K.unpack_table(buf)] == want


@pytest.mark.parametrize("rows", [2048, 50000])  # single-launch encode / two-pass encode (> 1024 tiles)
def test_output_capacity(ctx, oracle, rows):
    """An output buffer smaller than the packed call reports ERR_CAPACITY,
    writes nothing past the capacity, and leaves the context usable."""
    rng = np.random.default_rng(rows)
    xs = [(rng.standard_normal((rows, 16)) * 0.05).astype(np.float32) for _ in range(6)]
    jobs = [K.EncodeJob(dev(x), 0.01, t % 3) for t, x in enumerate(xs)]
    want = [oracle.encode_chunk(x.astype(np.float64).ravel(), 16, 0.01, t % 3) for t, x in enumerate(xs)]
    need = 4 + 16 * len(jobs) + sum(len(w) for w in want)
    cap = need // 2
    arena = torch.full((cap + 4096,), 0xA5, dtype=torch.uint8, device=DEV)
    cj = [j.to_c() for j in jobs]
    ctx.encode_raw(cj, K.LAYOUT_PACKED, arena[:cap])
    with pytest.raises(_lib.EmbcError) as e:
        ctx.sync()
    assert e.value.status == _lib.ERR_CAPACITY
    assert bool((arena[cap:] == 0xA5).all())
    out = torch.empty(need + 64, dtype=torch.uint8, device=DEV)
    ctx.encode_raw(cj, K.LAYOUT_PACKED, out)
    ctx.sync()
    buf = bytes(out[:need].cpu().numpy().tobytes())
    assert [buf[o:o + ln] for o, ln in K.unpack_table(buf)] == want


def test_empty_job_list(ctx, ref):
    """encode_chunks([]) + pack: the 4-byte rank count, written by the library
    (d_total included); the chunk and payload layouts are empty."""
    r = K.encode_chunks([], K.LAYOUT_PACKED)
    assert r.total == 4 and bytes(r.buffer.cpu().numpy().tobytes()) == ref.pack([])
    assert K.encode_chunks([], K.LAYOUT_CHUNKS).total == 0
    out = torch.full((8,), 0xAB, dtype=torch.uint8, device=DEV)
    tot = torch.full((1,), -1, dtype=torch.int64, device=DEV)
    ctx.encode_raw([], K.LAYOUT_PACKED, out, total=tot)
    ctx.sync()
    assert tot.item() == 4 and out.cpu().tolist() == [0, 0, 0, 0] + [0xAB] * 4
    with pytest.raises(_lib.EmbcError):
        ctx.encode_raw([], K.LAYOUT_PACKED, out[:2], total=tot)
