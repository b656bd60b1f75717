"""Dual-level adaptive error-bound controller (policy.hpp), host side.

Table-wise level: offline analysis classifies each table by the survival
ratio of its quantized lookup rows (policy.hpp:127-137, :188-193) and assigns
global_eb * alpha (large), global_eb (medium) or global_eb / beta (small)
(policy.hpp:95-102); a codec is chosen per table by Eq. 2
(policy.hpp:202-208, :239-274).  Iteration-wise level: the table's bound is
scaled by the stepwise / linear / logarithmic decay multiplier
(policy.hpp:308-342).

The arithmetic runs in the C ABI (embc_classify_table, embc_decay_multiplier,
embc_estimate_speedup: identical formulas, checked against the reference in
tests/test_capi.py); pattern counting (the embedding-vector analysis) runs on
the GPU (embc_pattern_counts).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import torch

from . import _lib
from . import codec as K

LARGE, MEDIUM, SMALL = 0, 1, 2
CLASS_NAMES = {LARGE: "large", MEDIUM: "medium", SMALL: "small"}
DECAY_FN = {"stepwise": 0, "linear": 1, "logarithmic": 2}


@dataclass
class DecayConfig:
    """policy.hpp:58-70."""
    function: str = "stepwise"
    start_scale: float = 1.0
    decay_end: int = 0
    step_count: int = 4


@dataclass
class PolicyConfig:
    """policy.hpp:75-103."""
    global_eb: float = 0.02
    alpha: float = 5.0 / 3.0
    beta: float = 3.0
    large_threshold: float = 0.70
    small_threshold: float = 0.95
    decay: DecayConfig = field(default_factory=DecayConfig)

    def eb_for(self, cls: int) -> float:
        if cls == LARGE:
            return self.global_eb * self.alpha
        if cls == SMALL:
            return self.global_eb / self.beta
        return self.global_eb


@dataclass
class ThroughputSample:
    """policy.hpp:107-112."""
    codec: int
    comp_bps: float
    decomp_bps: float
    ratio: float


@dataclass
class TableProfile:
    """policy.hpp:115-125."""
    table_id: int
    n_original_patterns: int = 0
    n_quantized_patterns: int = 0
    survival_ratio: float = 1.0
    homo_index: float = 0.0
    cls: int = MEDIUM
    codec: int = K.CODEC_RAW
    eb: float = 0.02
    measured: List[ThroughputSample] = field(default_factory=list)


def survival_ratio(n_original: int, n_quantized: int) -> float:
    if n_original == 0:
        raise _lib.CodecValueError("survival ratio needs a nonempty sample", status=_lib.ERR_VALUE)
    return float(n_quantized) / float(n_original)


def homo_index(n_original: int, n_quantized: int) -> float:
    return 1.0 - survival_ratio(n_original, n_quantized)


def classify_table(survival: float, cfg: PolicyConfig) -> int:
    cls, eb = C.c_int(), C.c_double()
    st = _lib.lib().embc_classify_table(survival, cfg.global_eb, cfg.alpha, cfg.beta, cfg.large_threshold,
                                        cfg.small_threshold, C.byref(cls), C.byref(eb))
    if st == _lib.ERR_CONFIG:
        raise _lib.CodecConfigError("invalid policy configuration", status=st)
    _lib.host_check(st, "embc_classify_table")
    return cls.value


def estimate_speedup(ratio: float, bandwidth: float, comp_bps: float, decomp_bps: float) -> float:
    out = C.c_double()
    st = _lib.lib().embc_estimate_speedup(ratio, bandwidth, comp_bps, decomp_bps, C.byref(out))
    if st == _lib.ERR_VALUE:
        raise _lib.CodecValueError("estimate_speedup arguments must all be positive", status=st)
    return out.value


def decay_multiplier(iteration: int, decay: DecayConfig) -> float:
    out = C.c_double()
    st = _lib.lib().embc_decay_multiplier(iteration, DECAY_FN[decay.function], decay.start_scale, decay.decay_end,
                                          decay.step_count, C.byref(out))
    if st == _lib.ERR_CONFIG:
        raise _lib.CodecConfigError("invalid decay configuration", status=st)
    _lib.host_check(st, "embc_decay_multiplier")
    return out.value


def eb_at(table_id: int, iteration: int, profiles: Dict[int, TableProfile], cfg: PolicyConfig) -> float:
    """policy.hpp:336-342."""
    base = profiles[table_id].eb if table_id in profiles else cfg.global_eb
    eb = base * decay_multiplier(iteration, cfg.decay)
    if not (eb > 0.0 and eb == eb and eb != float("inf")):
        raise _lib.CodecValueError(f"error bound must be finite and > 0, got {eb:f}", status=_lib.ERR_VALUE)
    return eb


# ---- profile persistence (config.hpp:247-303) --------------------------------

_CLASS_IDS = {v: k for k, v in CLASS_NAMES.items()}


def format_double(v: float) -> str:
    """detail::format_double (csv.hpp:31-37): std::to_chars shortest round-trip
    form -- the shorter of fixed and scientific notation, fixed on a tie."""
    from decimal import Decimal
    v = float(v)
    if v != v:
        return "nan" if repr(v)[0] != "-" else "-nan"
    if v in (float("inf"), float("-inf")):
        return "inf" if v > 0 else "-inf"
    sign = "-" if repr(v).startswith("-") else ""
    if v == 0.0:
        return sign + "0"
    t = Decimal(repr(abs(v))).normalize().as_tuple()
    digits = "".join(map(str, t.digits))
    point = len(digits) + t.exponent  # decimal point position after `point` digits
    if point <= 0:
        fixed = "0." + "0" * (-point) + digits
    elif point >= len(digits):  # an integer: to_chars spells out its exact digits (same length)
        fixed = str(int(abs(v)))
    else:
        fixed = digits[:point] + "." + digits[point:]
    se = point - 1
    sci = digits[0] + ("." + digits[1:] if len(digits) > 1 else "") + ("e-" if se < 0 else "e+") + f"{abs(se):02d}"
    return sign + (fixed if len(fixed) <= len(sci) else sci)


def write_profiles(path: str, profiles: Dict[int, TableProfile]) -> None:
    """write_profiles (config.hpp:247-271): the reference's key-value profile
    file, byte-identical for identical profiles."""
    lines = [f"profiles.count = {len(profiles)}"]
    for i, tid in enumerate(sorted(profiles)):
        p = profiles[tid]
        pre = f"profile.{i}."
        lines += [f"{pre}table = {tid}", f"{pre}n_original = {p.n_original_patterns}",
                  f"{pre}n_quantized = {p.n_quantized_patterns}", f"{pre}survival = {format_double(p.survival_ratio)}",
                  f"{pre}homo = {format_double(p.homo_index)}", f"{pre}class = {CLASS_NAMES[p.cls]}",
                  f"{pre}codec = {K.CODEC_NAMES[p.codec]}", f"{pre}eb = {format_double(p.eb)}"]
        for m in p.measured:
            mp = f"{pre}{K.CODEC_NAMES[m.codec]}."
            lines += [f"{mp}ratio = {format_double(m.ratio)}", f"{mp}comp_bps = {format_double(m.comp_bps)}",
                      f"{mp}decomp_bps = {format_double(m.decomp_bps)}"]
    with open(path, "w") as f:
        f.write("".join(line + "\n" for line in lines))


def _parse_kv(path: str) -> Dict[str, str]:
    """KeyValueConfig::parse_file (config.hpp:37-68)."""
    try:
        text = open(path).read()
    except OSError:
        raise _lib.CodecConfigError(f"cannot open config file '{path}'", status=_lib.ERR_CONFIG)
    kv: Dict[str, str] = {}
    for n, line in enumerate(text.split("\n"), 1):
        t = line.strip(" \t\r")
        if not t or t[0] == "#":
            continue
        if "=" not in t:
            raise _lib.CodecConfigError(f"{path}:{n}: expected 'key = value'", status=_lib.ERR_CONFIG)
        k, v = t.split("=", 1)
        k, v = k.strip(" \t\r"), v.strip(" \t\r")
        if not k:
            raise _lib.CodecConfigError(f"{path}:{n}: empty key", status=_lib.ERR_CONFIG)
        kv[k] = v
    return kv


def _kv_get(kv: Dict[str, str], key: str) -> str:
    if key not in kv:
        raise _lib.CodecConfigError(f"missing config key '{key}'", status=_lib.ERR_CONFIG)
    return kv[key]


def _kv_u64(kv, key) -> int:
    v = _kv_get(kv, key)
    if not v.isdigit():
        raise _lib.CodecConfigError(f"key '{key}' expects a non-negative integer, got '{v}'", status=_lib.ERR_CONFIG)
    return int(v)


def _kv_f64(kv, key) -> float:
    v = _kv_get(kv, key)
    try:
        if v.strip() != v or v.lower() in ("infinity", "-infinity") or "_" in v:
            raise ValueError
        return float(v)
    except ValueError:
        raise _lib.CodecConfigError(f"key '{key}' expects a number, got '{v}'", status=_lib.ERR_CONFIG)


def read_profiles(path: str) -> Dict[int, TableProfile]:
    """read_profiles (config.hpp:273-303)."""
    kv = _parse_kv(path)
    out: Dict[int, TableProfile] = {}
    for i in range(_kv_u64(kv, "profiles.count")):
        pre = f"profile.{i}."
        tid, no, nq = _kv_u64(kv, pre + "table"), _kv_u64(kv, pre + "n_original"), _kv_u64(kv, pre + "n_quantized")
        surv, homo = _kv_f64(kv, pre + "survival"), _kv_f64(kv, pre + "homo")
        cls_name = _kv_get(kv, pre + "class")
        if cls_name not in _CLASS_IDS:
            raise _lib.CodecConfigError(f"unknown table class '{cls_name}'", status=_lib.ERR_CONFIG)
        codec_name = _kv_get(kv, pre + "codec")
        if codec_name not in K.CODEC_IDS:
            raise _lib.CodecConfigError(f"unknown codec '{codec_name}'", status=_lib.ERR_CONFIG)
        p = TableProfile(tid, no, nq, surv, homo, _CLASS_IDS[cls_name], K.CODEC_IDS[codec_name],
                         _kv_f64(kv, pre + "eb"))
        for c in (K.CODEC_VLZ, K.CODEC_HUFFMAN):
            mp = f"{pre}{K.CODEC_NAMES[c]}."
            if mp + "ratio" in kv:
                p.measured.append(ThroughputSample(c, _kv_f64(kv, mp + "comp_bps"), _kv_f64(kv, mp + "decomp_bps"),
                                                   _kv_f64(kv, mp + "ratio")))
        out[p.table_id] = p
    return out


def _median_gpu_seconds(fn, runs: int = 5) -> float:
    """detail::median_seconds (policy.hpp:218-231) with CUDA events."""
    times = []
    for _ in range(runs):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        times.append(a.elapsed_time(b) / 1e3)
    times.sort()
    return max(times[runs // 2], 1e-9)


def select_codec(sample: torch.Tensor, eb: float, candidates: Sequence[int], bandwidth: float,
                 window: int = 255, timed: bool = True):
    """select_codec (policy.hpp:239-274) with the GPU codecs.  timed=False pins
    the choice to the compression ratio alone (Eq. 2 as bandwidth -> 0), which
    is deterministic; timed=True measures median-of-5 GPU throughputs as the
    reference does with wall clock."""
    if not candidates:
        raise _lib.CodecValueError("select_codec needs at least one candidate", status=_lib.ERR_VALUE)
    unc = float(sample.numel() * 4)
    measured = []
    best, best_ratio, chosen = -1.0, 0.0, K.CODEC_RAW
    for codec in candidates:
        job = K.EncodeJob(sample, eb, codec, window)
        r = K.encode_chunks([job], K.LAYOUT_CHUNKS)
        payload = r.total - K.HEADER_SIZE
        ratio = unc / payload
        if timed:
            ctx = K.Context.default()
            cj = [job.to_c()]
            out = torch.empty(r.total + 64, dtype=torch.uint8, device=sample.device)
            dec = torch.empty_like(sample)
            ref = _lib.ChunkRef()
            ref.offset, ref.length, ref.out = 0, r.total, dec.data_ptr()
            ref.dim, ref.count, ref.codec = sample.shape[1], sample.shape[0], codec
            comp_s = _median_gpu_seconds(lambda: ctx.encode_raw(cj, K.LAYOUT_CHUNKS, out))
            decomp_s = _median_gpu_seconds(lambda: ctx.decode_raw(r.buffer, [ref], K.OUT_F32, False))
            ctx.sync()
            m = ThroughputSample(codec, unc / comp_s, unc / decomp_s, ratio)
            speedup = estimate_speedup(ratio, bandwidth, m.comp_bps, m.decomp_bps)
        else:
            m = ThroughputSample(codec, float("inf"), float("inf"), ratio)
            speedup = ratio
        measured.append(m)
        if best < 0.0 or speedup > best or (speedup == best and codec < chosen):
            best, best_ratio, chosen = speedup, ratio, codec
    if best_ratio <= 1.0:
        chosen = K.CODEC_RAW
    return chosen, measured


def offline_analysis(samples: Dict[int, torch.Tensor], cfg: PolicyConfig, bandwidth: float,
                     window: int = 255, timed: bool = False) -> Dict[int, TableProfile]:
    """offline_analysis (policy.hpp:278-302): one profile per sampled table."""
    profiles = {}
    for tid, sample in samples.items():
        p = TableProfile(tid)
        o, q = K.pattern_counts(sample, cfg.global_eb)
        p.n_original_patterns, p.n_quantized_patterns = o, q
        p.survival_ratio = survival_ratio(o, q)
        p.homo_index = homo_index(o, q)
        p.cls = classify_table(p.survival_ratio, cfg)
        p.eb = cfg.eb_for(p.cls)
        p.codec, p.measured = select_codec(sample, p.eb, [K.CODEC_VLZ, K.CODEC_HUFFMAN], bandwidth, window, timed)
        profiles[tid] = p
    return profiles
