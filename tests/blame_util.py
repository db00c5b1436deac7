"""Helpers for the f4 tests: build trace sets from the golden line lists, and an
independent 1-ns brute force (exact rationals) of GPU-idleness blame."""
from fractions import Fraction

import numpy as np

NONE = 0xFFFFFFFF


def from_lines(cases):
    """cases: list of (n_routines, lines) per scope -> trace-set dict."""
    lo, kind, scope, t, c = [0], [], [], [], []
    n_routines = max(n for n, _ in cases)
    for s, (_, lines) in enumerate(cases):
        for k, ev in lines:
            kind.append(0 if k == "gpu" else 1)
            scope.append(s)
            t += [int(x[0]) for x in ev]
            c += [NONE if x[1] is None else int(x[1]) for x in ev]
            lo.append(len(t))
    return dict(line_off=np.array(lo, np.uint64), line_kind=np.array(kind, np.uint8),
                line_scope=np.array(scope, np.uint32), time=np.array(t, np.uint64),
                ctx=np.array(c, np.uint32), n_scopes=len(cases), n_routines=n_routines)


def brute_force(tr):
    """Per scope and per nanosecond: state of each line = ctx of its last change point <= t
    (idle before the first and from the last one on); returns exact num, total, gpu_idle and
    Fraction blame per (scope, routine)."""
    lo, kind, scope = tr["line_off"].astype(np.int64), tr["line_kind"], tr["line_scope"]
    T, C = tr["time"].astype(np.int64), tr["ctx"]
    S, R = tr["n_scopes"], tr["n_routines"]
    num, total, idle = {}, [0] * S, [0] * S
    blame = [[Fraction(0)] * R for _ in range(S)]
    for s in range(S):
        lines = [l for l in range(len(kind)) if scope[l] == s]
        ts = [int(T[e]) for l in lines for e in range(lo[l], lo[l + 1])]
        for t in range(min(ts), max(ts)):
            gpu_busy, active = False, []
            for l in lines:
                ev = [e for e in range(lo[l], lo[l + 1]) if T[e] <= t]
                if not ev or ev[-1] == lo[l + 1] - 1 or C[ev[-1]] == NONE:
                    continue
                if kind[l] == 0:
                    gpu_busy = True
                else:
                    active.append(int(C[ev[-1]]))
            if gpu_busy:
                continue
            idle[s] += 1
            if not active:
                continue
            total[s] += 1
            for r in active:
                num[(s, r, len(active))] = num.get((s, r, len(active)), 0) + 1
                blame[s][r] += Fraction(1, len(active))
    return num, total, idle, blame


def random_trace(rng, scopes, max_lines=(4, 5), t_max=60, max_events=9):
    cases = []
    R = int(rng.integers(1, 5))
    for _ in range(scopes):
        lines = []
        n_gpu, n_cpu = int(rng.integers(1, max_lines[0])), int(rng.integers(0, max_lines[1]))
        kinds = ["gpu"] * n_gpu + ["cpu"] * n_cpu
        rng.shuffle(kinds)
        for k in kinds:
            m = int(rng.integers(1, max_events))
            ts = np.sort(rng.integers(0, t_max, m))
            ev = []
            for t in ts:
                idle = rng.random() < 0.4
                ev.append([int(t), None if idle else int(rng.integers(0, R if k == "cpu" else 9))])
            lines.append([k, ev])
        cases.append((R, lines))
    return from_lines(cases)
