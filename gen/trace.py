"""Seeded synthetic trace sets for f4 (GPU-idleness blame, §6.2).

Shared by the oracle tests and the GPU path; holds none of the method's arithmetic.  A trace
set is a dict of numpy arrays: line_off u64 [L+1] (CSR over events), line_kind u8 [L] (0 GPU
stream, 1 CPU thread), line_scope u32 [L] (rank; non-decreasing), time u64 [E], ctx u32 [E]
(GPU: kernel id, CPU: routine id at the attribution depth, NONE = idle), n_scopes, n_routines.

Model ("trace recipe"): each rank alternates host phases (CPU threads run
routines, GPU streams idle) and device phases (each stream runs a burst of kernels with
gaps; the main CPU thread waits in routine 0 = "sync").  Phase lengths are lognormal; GPU
bursts spill into the preceding host phase and CPU work spills into the device phase with
some probability, so idle periods partially overlap CPU activity (the cases blame splits).
Timestamps are absolute 64-bit nanoseconds (epoch-sized base)."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

NONE = 0xFFFFFFFF


@dataclass(frozen=True)
class TraceConfig:
    name: str
    scopes: int
    gpu_lines: int
    cpu_lines: int
    iters: int
    kernels_per_phase: int
    segs_per_phase: int
    n_routines: int
    n_kernels: int
    seed: int


TRACE_CONFIGS = {
    "B1": TraceConfig("B1", 3, 2, 3, 12, 3, 2, 20, 5, 601),
    "B2": TraceConfig("B2", 8, 6, 8, 300, 16, 4, 200, 50, 602),
    "B3": TraceConfig("B3", 64, 6, 8, 2000, 16, 4, 500, 50, 603),
}


def _zipf(rng, n, size):
    w = 1.0 / np.arange(1, n + 1) ** 1.1
    return rng.choice(n, size=size, p=w / w.sum()).astype(np.uint32)


def _alternate(rng, lo, hi, pairs, ids):
    """Sorted change points in [lo, hi) per row: 2*pairs uniforms, ctx alternating id / NONE."""
    u = np.sort(rng.random((len(lo), 2 * pairs)), axis=1)
    t = lo[:, None] + u * (hi - lo)[:, None]
    c = np.full(t.shape, NONE, np.uint32)
    c[:, 0::2] = ids.reshape(len(lo), pairs)
    return t, c


def trace_set(cfg: TraceConfig | str) -> dict:
    if isinstance(cfg, str):
        cfg = TRACE_CONFIGS[cfg]
    rng = np.random.default_rng(cfg.seed)
    times, ctxs, kinds, scopes, lens = [], [], [], [], []
    base = np.uint64(1_700_000_000_000_000_000)
    for s in range(cfg.scopes):
        I = cfg.iters
        lc = rng.lognormal(np.log(20_000), 0.6, I)              # host phase, ns
        lg = rng.lognormal(np.log(150_000), 0.5, I)             # device phase, ns
        start = rng.uniform(0, 1e6) + np.concatenate([[0], np.cumsum(lc + lg)[:-1]])
        gstart = start + lc
        order = rng.permutation(cfg.gpu_lines + cfg.cpu_lines)   # kinds interleaved within a rank
        for li in order:
            if li < cfg.gpu_lines:
                spill = np.where(rng.random(I) < 0.3, rng.uniform(0, 0.3, I) * lc, 0.0)
                keep = rng.random(I) < 0.92
                lo, hi = (gstart - spill)[keep], (gstart + lg)[keep]
                t, c = _alternate(rng, lo, hi, cfg.kernels_per_phase,
                                  _zipf(rng, cfg.n_kernels, keep.sum() * cfg.kernels_per_phase))
                kind = 0
            else:
                main = li == cfg.gpu_lines
                hi = gstart + np.where(rng.random(I) < 0.4, 0.2 * lg, 0.0)
                t, c = _alternate(rng, start, hi, cfg.segs_per_phase,
                                  1 + _zipf(rng, cfg.n_routines - 1, I * cfg.segs_per_phase))
                if main:   # the main thread waits in routine 0 ("sync") for the device phase
                    ts = np.stack([np.maximum(t[:, -1], hi), gstart + lg], 1)
                    t = np.concatenate([t, ts], 1)
                    c = np.concatenate([c, np.stack([np.zeros(I, np.uint32), np.full(I, NONE, np.uint32)], 1)], 1)
                kind = 1
            t = t.reshape(-1)
            c = c.reshape(-1)
            times.append(base + np.floor(t).astype(np.uint64))
            ctxs.append(c)
            kinds.append(kind)
            scopes.append(s)
            lens.append(len(t))
    return dict(line_off=np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64),
                line_kind=np.array(kinds, np.uint8), line_scope=np.array(scopes, np.uint32),
                time=np.concatenate(times), ctx=np.concatenate(ctxs).astype(np.uint32),
                n_scopes=cfg.scopes, n_routines=cfg.n_routines)
