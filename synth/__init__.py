"""Seeded synthetic workloads for the Sprout hot path (inputs only).

This module builds the INPUTS of the method -- carbon-intensity traces,
per-segment request counts, Llama2-shaped generated-token tables, opt-out and
model-class flags, the level profiles e, p and the preference vectors q -- and
nothing of the method's arithmetic (no LP, no selection, no carbon
accounting).  It is the only module shared by the oracle side (tests, bench
cpu_baseline) and the CUDA side (bench, binding tests).

The token generator is counter-based (Philox4x32-10 on stream 1, one call per
global request index) with integer quantile / ratio tables, so that the same
request can be regenerated bit-exactly anywhere: by ``gen_tokens`` here
(numpy) and by the harness-only device kernel ``sprout_generate_trace``.  The
selection draw (stream 0) is NOT generated here: the oracle and the CUDA path
each implement it (reading L10 in DESIGN.md).

Recipe; paper anchors:
  * regions TX/CA/SA/NL/GB and their annual min/max CI: Table II;
  * q = [0.5, 0.3, 0.2] for TX: P:190;
  * PUE 1.2: P:153; T_life = 5 years: P:54;
  * energy/time linear in generated tokens: P:87-98 (Fig. motiv1(b));
  * directive levels L1/L2 cut generated tokens.
Everything else (sinusoid + AR(1) CI shape, diurnal arrivals, lognormal
token lengths, the per-token coefficients, CO2_embed = 150 kg) is synthetic.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

# --------------------------------------------------------------------------
# containers


@dataclasses.dataclass
class Problem:
    """The LP grid of Eqs. 2-7 over regions x intervals x xi."""
    n: int                  # directive levels
    R: int                  # regions
    T: int                  # CI intervals per region
    X: int                  # quality coefficients xi
    k0: np.ndarray          # [R*T] gCO2/kWh
    kmin: np.ndarray        # [R]
    kmax: np.ndarray        # [R]
    xi: np.ndarray          # [X] paper xi (allowed deviation)
    e: np.ndarray           # [R][n] (or [R*T][n]) kWh per request at each level
    p: np.ndarray           # [R][n] (or [R*T][n]) seconds per request
    q: np.ndarray           # [R][n] (or [R*T][n]) preference rates
    profile_per_interval: int
    k1: float               # gCO2/s embodied rate
    pue: float

    @property
    def S(self) -> int:
        return self.R * self.T

    @property
    def C(self) -> int:
        return self.R * self.T * self.X


@dataclasses.dataclass
class CostModel:
    """Per-request energy/time model E = ef + et*tok, T = pf + pt*tok per
    (class, level) (reading L11) and the selection seed."""
    seed: int
    n_classes: int
    ef: np.ndarray   # [4][8] kWh
    et: np.ndarray   # [4][8] kWh / token
    pf: np.ndarray   # [4][8] s
    pt: np.ndarray   # [4][8] s / token


@dataclasses.dataclass
class TraceSpec:
    """How requests are laid out and how their tokens/flags are generated."""
    seg_offsets: np.ndarray  # [S+1] int64, global request index of each segment start
    gen_seed: int
    n_levels: int
    n_classes: int
    has_flags: bool
    pin_thresh: int          # pinned iff (w3 & 0xFFFFFF) < pin_thresh
    q0_table: np.ndarray     # [n_classes][4096] uint16
    ratio_table: np.ndarray  # [8][256] uint16 (row 0 unused)

    @property
    def N(self) -> int:
        return int(self.seg_offsets[-1])


@dataclasses.dataclass
class Workload:
    name: str
    prob: Problem
    cost: CostModel
    spec: TraceSpec
    description: str = ""

    @property
    def N(self) -> int:
        return self.spec.N


# --------------------------------------------------------------------------
# Philox4x32-10 (Random123 constants), numpy-vectorised, used here ONLY for
# the input generator's stream 1.

_M0 = np.uint64(0xD2511F53)
_M1 = np.uint64(0xCD9E8D57)
_W0 = 0x9E3779B9
_W1 = 0xBB67AE85
_MASK = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0: int, k1: int):
    c0 = np.asarray(c0, np.uint64) & _MASK
    c1 = np.asarray(c1, np.uint64) & _MASK
    c2 = np.asarray(c2, np.uint64) & _MASK
    c3 = np.asarray(c3, np.uint64) & _MASK
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    ka, kb = k0 & 0xFFFFFFFF, k1 & 0xFFFFFFFF
    for rnd in range(10):
        if rnd:
            ka = (ka + _W0) & 0xFFFFFFFF
            kb = (kb + _W1) & 0xFFFFFFFF
        p0 = c0 * _M0
        p1 = c2 * _M1
        n0 = (p1 >> np.uint64(32)) ^ c1 ^ np.uint64(ka)
        n1 = p1 & _MASK
        n2 = (p0 >> np.uint64(32)) ^ c3 ^ np.uint64(kb)
        n3 = p0 & _MASK
        c0, c1, c2, c3 = n0, n1, n2, n3
    return (c0.astype(np.uint32), c1.astype(np.uint32), c2.astype(np.uint32), c3.astype(np.uint32))


GEN_STREAM = 1  # counter word 2 of the generator's Philox calls


def gen_tokens(spec: TraceSpec, g_lo: int, g_hi: int):
    """Generated tokens [n][g_hi-g_lo] uint16 and flags [g_hi-g_lo] uint8 (or
    None) of global requests [g_lo, g_hi).  One Philox call per request:
    ctr = (g lo32, g hi32, 1, 0), key = gen_seed.  Integer tables only."""
    n = spec.n_levels
    g = np.arange(g_lo, g_hi, dtype=np.uint64)
    w0, w1, w2, w3 = philox4x32_10(g & _MASK, g >> np.uint64(32), GEN_STREAM, 0,
                                   spec.gen_seed & 0xFFFFFFFF, (spec.gen_seed >> 32) & 0xFFFFFFFF)
    NC = spec.n_classes
    cls = ((w3.astype(np.uint64) >> np.uint64(16)) * np.uint64(NC)) >> np.uint64(16)
    cls = cls.astype(np.int64)
    tok0 = spec.q0_table[cls, (w0 >> np.uint32(20)).astype(np.int64)].astype(np.uint32)
    toks = np.empty((n, g.size), np.uint16)
    toks[0] = tok0
    for i in range(1, n):
        src = w1 if i <= 4 else w2
        sh = 8 * (i - 1) if i <= 4 else 8 * (i - 5)
        b = ((src >> np.uint32(sh)) & np.uint32(0xFF)).astype(np.int64)
        t = (tok0 * spec.ratio_table[i, b].astype(np.uint32)) >> np.uint32(16)
        toks[i] = np.maximum(t, 1).astype(np.uint16)
    flags = None
    if spec.has_flags:
        pinned = ((w3 & np.uint32(0xFFFFFF)) < np.uint32(spec.pin_thresh)).astype(np.uint8)
        flags = (pinned | (cls.astype(np.uint8) << np.uint8(1))).astype(np.uint8)
    return toks, flags


# --------------------------------------------------------------------------
# the paper-shaped regions (Table II) and q vectors

REGIONS = ["TX", "CA", "SA", "NL", "GB"]
TABLE2 = {"TX": (124.0, 494.0), "CA": (55.0, 331.0), "SA": (10.0, 526.0),
          "NL": (23.0, 463.0), "GB": (24.0, 282.0)}
Q3 = {"TX": [0.5, 0.3, 0.2],
      "CA": [0.45, 0.33, 0.22],
      "SA": [0.40, 0.35, 0.25],
      "NL": [0.55, 0.28, 0.17],
      "GB": [0.34, 0.36, 0.30]}       # L1-preferred period

PUE = 1.2
T_LIFE_S = 5 * 365 * 86400
CO2_EMBED_G = 150_000.0                     # reading L14 (synthetic)
K1 = CO2_EMBED_G / T_LIFE_S                 # gCO2/s
BASE_SEED = 0x5350524F5554


def ci_trace(rng: np.random.Generator, T: int, per_day: int, kmin: float, kmax: float,
             phase_h: float) -> np.ndarray:
    """Min-max normalised diurnal + seasonal + AR(1) shape scaled to
    [kmin, kmax]; min and max are attained exactly (Table II bounds)."""
    t = np.arange(T, dtype=np.float64)
    hours = t * (24.0 / per_day)
    day = hours / 24.0
    diurnal = np.cos(2 * np.pi * (hours - phase_h) / 24.0)
    seasonal = 0.5 * np.sin(2 * np.pi * day / 365.0 + rng.uniform(0, 2 * np.pi))
    from scipy.signal import lfilter
    phi = 0.9 ** (24.0 / per_day)            # AR(1) coefficient 0.9 per hour
    eps = rng.normal(0.0, 0.35 * math.sqrt(1 - phi * phi), size=T)
    ar = lfilter([1.0], [1.0, -phi], eps)
    raw = diurnal + seasonal + ar
    span = raw.max() - raw.min()
    s = (raw - raw.min()) / span if span > 0 else np.zeros(T)
    return kmin + (kmax - kmin) * s


def largest_remainder(total: int, weights: np.ndarray) -> np.ndarray:
    w = np.asarray(weights, dtype=np.float64)
    quota = total * w / w.sum()
    base = np.floor(quota).astype(np.int64)
    rem = total - int(base.sum())
    if rem > 0:
        order = np.argsort(-(quota - base), kind="stable")
        base[order[:rem]] += 1
    return base


def arrivals(N: int, R: int, T: int, per_day: int) -> np.ndarray:
    """Per-(region, interval) request counts, diurnal weights
    1 + 0.6 sin(2 pi (h - 14)/24), equal region shares, sum exactly N."""
    per_region = largest_remainder(N, np.ones(R))
    hours = np.arange(T, dtype=np.float64) * (24.0 / per_day)
    w = 1.0 + 0.6 * np.sin(2 * np.pi * (hours - 14.0) / 24.0)
    m = np.concatenate([largest_remainder(int(per_region[r]), w) for r in range(R)])
    return m


def q0_table(mean_tokens: float, sigma: float = 0.8) -> np.ndarray:
    """4096-entry quantile table of a lognormal output length, clipped to
    [1, 4095] (Llama2's 4096-token context)."""
    from scipy.special import ndtri
    mu = math.log(mean_tokens) - 0.5 * sigma * sigma
    u = (np.arange(4096, dtype=np.float64) + 0.5) / 4096.0
    v = np.exp(mu + sigma * ndtri(u))
    return np.clip(np.rint(v), 1, 4095).astype(np.uint16)


def ratio_table(ratios) -> np.ndarray:
    """[8][256] fixed-point (x 2^-16) per-level length ratios vs L0, mean
    ratio rho_i, spread uniformly over [0.5, 1.5) * rho_i."""
    tab = np.zeros((8, 256), np.uint16)
    k = (np.arange(256, dtype=np.float64) + 0.5) / 256.0
    for i, rho in enumerate(ratios):
        if i == 0:
            continue
        tab[i] = np.clip(np.rint(65536.0 * rho * (0.5 + k)), 1, 65535).astype(np.uint16)
    return tab


def class_shares(NC: int) -> np.ndarray:
    v = np.arange(65536, dtype=np.uint64)
    c = (v * np.uint64(NC)) >> np.uint64(16)
    return np.bincount(c.astype(np.int64), minlength=NC).astype(np.float64) / 65536.0


def level_means(spec: TraceSpec) -> np.ndarray:
    """Exact mean generated tokens per (class, level) of the generator
    (enumerating all 4096 x 256 table pairs; integer sums, one division)."""
    n, NC = spec.n_levels, spec.n_classes
    mu = np.zeros((NC, n))
    for c in range(NC):
        q0 = spec.q0_table[c].astype(np.int64)
        mu[c, 0] = float(q0.sum()) / 4096.0
        for i in range(1, n):
            t = (q0[:, None] * spec.ratio_table[i][None, :].astype(np.int64)) >> 16
            t = np.maximum(t, 1)
            mu[c, i] = float(t.sum()) / (4096.0 * 256.0)
    return mu


def cost_coefficients(NC: int, n: int):
    """A100-like per-request energy/time coefficients (synthetic; reading L11).
    Class 0 = Llama2-13B, class 1 = Llama2-7B (0.55x energy, 0.6x time).
    A directive adds a few prefill tokens: +2% fixed cost for L>0."""
    ef = np.zeros((4, 8)); et = np.zeros((4, 8)); pf = np.zeros((4, 8)); pt = np.zeros((4, 8))
    base = [(2.0e-6, 1.0e-7, 0.01, 0.0016), (1.1e-6, 0.55e-7, 0.006, 0.00096)]
    for c in range(NC):
        b = base[c % 2]
        for L in range(n):
            bump = 1.0 if L == 0 else 1.02
            ef[c, L] = b[0] * bump
            et[c, L] = b[1]
            pf[c, L] = b[2] * bump
            pt[c, L] = b[3]
    return ef, et, pf, pt


def profiles(spec: TraceSpec, ef, et, pf, pt) -> tuple[np.ndarray, np.ndarray]:
    """e_i, p_i: the average energy / time per request at level i
    under the generator, computed exactly from level_means (reading L12)."""
    mu = level_means(spec)
    sh = class_shares(spec.n_classes)
    n = spec.n_levels
    e = np.zeros(n); p = np.zeros(n)
    for i in range(n):
        for c in range(spec.n_classes):
            e[i] += sh[c] * (ef[c, i] + et[c, i] * mu[c, i])
            p[i] += sh[c] * (pf[c, i] + pt[c, i] * mu[c, i])
    return e, p


# --------------------------------------------------------------------------
# the five BASELINE.json configurations (SURVEY 8, table "Config")

CONFIGS = ["C1", "C2", "C3", "C4", "C5"]


def make_workload(name: str, n_requests: Optional[int] = None, n_intervals: Optional[int] = None,
                  n_regions: Optional[int] = None, xi: Optional[np.ndarray] = None,
                  seed_offset: int = 0) -> Workload:
    """Build one of C1..C5 (optionally scaled down for tests).

    Reading L1: the configs' "xi = 0.9" / "{0.8, 0.9, 0.95}" are the quality
    CRITERION tau = 1 - xi of P:195 ("at least 90% as favorable"); the paper's
    xi is 1 - tau.  The 64-value sweep of C4 is xi_k = k/63."""
    idx = CONFIGS.index(name) if name in CONFIGS else 9
    seed = BASE_SEED + idx + seed_offset
    rng = np.random.default_rng(seed)
    if name == "C1":
        n, R, per_day, T, N, xis, NC, flags = 3, 1, 24, 24, 1000, [0.1], 1, True
    elif name == "C2":
        n, R, per_day, T, N, xis, NC, flags = 3, 5, 24, 8760, 10**6, [0.2, 0.1, 0.05], 1, True
    elif name == "C3":
        n, R, per_day, T, N, xis, NC, flags = 3, 5, 288, 105120, 10**8, [0.1], 2, True
    elif name == "C4":
        n, R, per_day, T, N, xis, NC, flags = 3, 5, 24, 8760, 10**9, list(np.arange(64) / 63.0), 1, False
    elif name == "C5":
        n, R, per_day, T, N, xis, NC, flags = 5, 256, 24, 8760, 10**10, [0.1], 1, False
    else:
        raise ValueError(name)
    if n_requests is not None:
        N = int(n_requests)
    if n_intervals is not None:
        T = int(n_intervals)
    if n_regions is not None:
        R = int(n_regions)
    if xi is not None:
        xis = list(xi)
    X = len(xis)

    # carbon-intensity traces
    k0 = np.empty(R * T)
    kmin = np.empty(R)
    kmax = np.empty(R)
    q = np.empty((R, n))
    if name == "C5":
        lo = rng.uniform(5.0, 150.0, size=R)
        hi = lo + rng.uniform(100.0, 600.0, size=R)
        for r in range(R):
            k0[r * T:(r + 1) * T] = ci_trace(rng, T, per_day, float(lo[r]), float(hi[r]), rng.uniform(0, 24))
            kmin[r], kmax[r] = lo[r], hi[r]
            q[r] = rng.dirichlet(np.full(n, 2.0))
    else:
        for r in range(R):
            reg = REGIONS[2] if name == "C1" else REGIONS[r % 5]
            lo, hi = TABLE2[reg]
            # C1 = the first 24 h of an SA year; its kmin/kmax are those of
            # the 24 replayed values (reading L4), so f spans exactly [0, 1].
            full = ci_trace(rng, 8760 if name == "C1" else T, per_day, lo, hi, 13.0 + 2.0 * (r % 5))
            trace = full[:T]
            k0[r * T:(r + 1) * T] = trace
            kmin[r], kmax[r] = trace.min(), trace.max()
            q[r] = Q3[reg] if n == 3 else rng.dirichlet(np.full(n, 2.0))

    # requests
    m = arrivals(N, R, T, per_day)
    seg_offsets = np.zeros(R * T + 1, np.int64)
    np.cumsum(m, out=seg_offsets[1:])

    if n == 3:
        ratios = [1.0, 1.0 / 3.0, 1.0 / 5.0]
    else:
        ratios = [1.0 / (i + 1) for i in range(n)]
    means = [250.0, 220.0][:NC]
    spec = TraceSpec(seg_offsets=seg_offsets, gen_seed=(seed * 0x9E3779B97F4A7C15 + 1) & ((1 << 64) - 1),
                     n_levels=n, n_classes=NC, has_flags=flags, pin_thresh=167772 if flags else 0,
                     q0_table=np.stack([q0_table(mu) for mu in means]), ratio_table=ratio_table(ratios))
    ef, et, pf, pt = cost_coefficients(NC, n)
    e, p = profiles(spec, ef, et, pf, pt)
    prob = Problem(n=n, R=R, T=T, X=X, k0=k0, kmin=kmin, kmax=kmax, xi=np.asarray(xis, np.float64),
                   e=np.tile(e, (R, 1)), p=np.tile(p, (R, 1)), q=np.ascontiguousarray(q),
                   profile_per_interval=0, k1=K1, pue=PUE)
    cost = CostModel(seed=(seed ^ 0x5E1EC7105EED) & ((1 << 64) - 1), n_classes=NC, ef=ef, et=et, pf=pf, pt=pt)
    return Workload(name=name, prob=prob, cost=cost, spec=spec,
                    description=f"{name}: R={R} T={T} n={n} X={X} N={N} classes={NC} flags={flags}")


# --------------------------------------------------------------------------
# sharding: contiguous segment ranges, split where the prefix
# request count crosses k*N/G.  The local request buffer starts at the
# rank's first global request rounded down to a multiple of 8 (the C-ABI's
# alignment rule for first_request); requests before the first segment are
# padding and belong to no segment.

@dataclasses.dataclass
class Shard:
    rank: int
    world: int
    first_segment: int
    n_segments: int
    first_request: int      # global index of local request 0 (multiple of 8)
    n_requests: int         # local requests, including the leading padding
    seg_offsets: np.ndarray  # [n_segments+1] local offsets


def shard(spec: TraceSpec, world: int, rank: int) -> Shard:
    off = spec.seg_offsets
    S = off.size - 1
    N = int(off[-1])
    cuts = [0] + [int(np.searchsorted(off[:-1], (k * N) // world, side="left")) for k in range(1, world)] + [S]
    cuts = [min(max(c, 0), S) for c in cuts]
    for k in range(1, len(cuts)):
        cuts[k] = max(cuts[k], cuts[k - 1])
    s_lo, s_hi = cuts[rank], cuts[rank + 1]
    g_lo, g_hi = int(off[s_lo]), int(off[s_hi])
    base = (g_lo // 8) * 8
    local = (off[s_lo:s_hi + 1] - base).astype(np.int64)
    return Shard(rank=rank, world=world, first_segment=s_lo, n_segments=s_hi - s_lo,
                 first_request=base, n_requests=g_hi - base, seg_offsets=local)


def shard_regions(spec: TraceSpec, T: int, world: int, rank: int) -> Shard:
    """Contiguous whole regions per rank (closed-loop chains are per region):
    regions [rank*R/world, (rank+1)*R/world)."""
    off = spec.seg_offsets
    R = (off.size - 1) // T
    r_lo, r_hi = (rank * R) // world, ((rank + 1) * R) // world
    s_lo, s_hi = r_lo * T, r_hi * T
    g_lo, g_hi = int(off[s_lo]), int(off[s_hi])
    base = (g_lo // 8) * 8
    local = (off[s_lo:s_hi + 1] - base).astype(np.int64)
    return Shard(rank=rank, world=world, first_segment=s_lo, n_segments=s_hi - s_lo,
                 first_request=base, n_requests=g_hi - base, seg_offsets=local)


def pitch_for(n_requests: int) -> int:
    """Token-plane pitch: a multiple of 8 u16 (16 B) covering n_requests."""
    return max(8, ((n_requests + 7) // 8) * 8)


def host_trace(spec: TraceSpec, sh: Shard):
    """Host-generated local trace of a shard: tokens [n][pitch] u16 (zero
    padded beyond n_requests) and flags [pitch] u8 or None."""
    pitch = pitch_for(sh.n_requests)
    toks = np.zeros((spec.n_levels, pitch), np.uint16)
    t, f = gen_tokens(spec, sh.first_request, sh.first_request + sh.n_requests)
    toks[:, :sh.n_requests] = t
    flags = None
    if f is not None:
        flags = np.zeros(pitch, np.uint8)
        flags[:sh.n_requests] = f
    return toks, flags


def sample_segments(spec: TraceSpec, first_segment: int, n_segments: int, every: int = 97) -> np.ndarray:
    """Deterministic segment sample: every `every`-th segment
    plus the first, the last and the largest of the range."""
    off = spec.seg_offsets
    ids = set(range(first_segment, first_segment + n_segments, every))
    if n_segments:
        ids.add(first_segment)
        ids.add(first_segment + n_segments - 1)
        m = np.diff(off[first_segment:first_segment + n_segments + 1])
        ids.add(first_segment + int(np.argmax(m)))
    return np.array(sorted(ids), np.int64)
