"""The reference's training-schedule simulator (Simulator::run_schedule,
commsim.hpp:200-266) with the codec on the GPU (embc_simulate in
csrc/simulate.cpp): R ranks, one forward all-to-all per iteration, each
rank's table compressed per destination, packed, unpacked and decoded by the
sm_100a kernels.  Byte accounting, delivered-value digests and
SimReport::deterministic_digest (commsim.hpp:146-163) are the reference's; the
comp/decomp times are device-measured.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Sequence

from . import _lib
from . import policy as P

_DECAY_FN = {"stepwise": 0, "linear": 1, "log": 2}


@dataclass
class SimConfig:
    """SimConfig (commsim.hpp:30-62)."""
    ranks: int = 4
    batch: int = 128
    iterations: int = 100
    seed: int = 1
    compression: bool = True
    bandwidth: float = 4e9
    latency: float = 20e-6
    policy: P.PolicyConfig = field(default_factory=P.PolicyConfig)
    tables: List[tuple] = field(default_factory=list)  # (rows, dim, dist, mu, sigma, lo, hi, zipf)


@dataclass
class IterationStats:
    """IterationStats (commsim.hpp:77-96)."""
    iteration: int
    eb_max: float
    uncompressed_bytes: int
    payload_bytes: int
    metadata_bytes: int
    wire_bytes: int
    comp_time: float
    decomp_time: float
    max_abs_error: float
    delivery_conserved: bool
    delivered_digest: int


@dataclass
class SimReport:
    ranks: int
    batch: int
    compression: bool
    iterations: List[IterationStats]
    deterministic_digest: int

    def compression_ratio(self, begin: int = 0, end: int = 1 << 62) -> float:
        """SimReport::compression_ratio (commsim.hpp:133-142)."""
        unc = sum(it.uncompressed_bytes for it in self.iterations if begin <= it.iteration < end)
        pay = sum(it.payload_bytes for it in self.iterations if begin <= it.iteration < end)
        return 1.0 if pay == 0 else unc / pay


def run_training_schedule(cfg: SimConfig, profiles: Dict[int, P.TableProfile], device: int = 0) -> SimReport:
    """run_training_schedule (commsim.hpp:505-508)."""
    L = _lib.lib()
    c = _lib.SimConfig()
    c.ranks, c.batch, c.iterations, c.compression = cfg.ranks, cfg.batch, cfg.iterations, int(cfg.compression)
    c.seed, c.global_eb = cfg.seed, cfg.policy.global_eb
    d = cfg.policy.decay
    c.decay_fn, c.decay_steps, c.decay_start_scale, c.decay_end = _DECAY_FN[d.function], d.step_count, \
        d.start_scale, d.decay_end
    if not cfg.tables:
        raise _lib.CodecConfigError("at least one table spec is required", status=_lib.ERR_CONFIG)
    tabs = (_lib.SimTable * len(cfg.tables))()
    for i, t in enumerate(cfg.tables):
        rows, dim, dist, mu, sigma, lo, hi, zipf = t
        tabs[i].rows, tabs[i].dim, tabs[i].dist = rows, dim, dist
        tabs[i].mu, tabs[i].sigma, tabs[i].lo, tabs[i].hi, tabs[i].zipf_s = mu, sigma, lo, hi, zipf
    R = cfg.ranks
    codec = (C.c_uint8 * R)(*[profiles[r].codec if r in profiles else _lib.CODEC_RAW for r in range(R)])
    ebs = (C.c_double * R)(*[profiles[r].eb if r in profiles else cfg.policy.global_eb for r in range(R)])
    out = (_lib.SimIteration * max(1, cfg.iterations))()
    rep = C.c_uint64()
    err = _lib.EmbcErrorRec()
    st = L.embc_simulate(device, C.byref(c), tabs, len(cfg.tables), codec, ebs, out, C.byref(rep), C.byref(err))
    if st != _lib.OK:
        _lib.raise_for(st, err.message.decode(errors="replace"), err.reason)
    its = [IterationStats(o.iteration, o.eb_max, o.uncompressed_bytes, o.payload_bytes, o.metadata_bytes,
                          o.wire_bytes, o.comp_time, o.decomp_time, o.max_abs_error, bool(o.delivery_conserved),
                          o.delivered_digest) for o in out[:cfg.iterations]]
    return SimReport(R, cfg.batch, cfg.compression, its, rep.value)


def report_rows(rep: SimReport) -> Sequence[dict]:
    return [vars(it) for it in rep.iterations]
