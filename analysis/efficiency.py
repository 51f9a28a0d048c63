"""The paper's speedup/efficiency model (§1.3-§3, Eqs. 1-15), and its
application to this build's measured c4 batching sweep.

Equation numbers are the paper's:
  (1) S_p = T_1 / T_p                      (2) E_p = S_p / p
  (3) T_p = [(1 - a) + a/p] T_1            (4) S_p = p / (p - a (p - 1))   (Amdahl)
  (5) E_p = 1 / ((1 - a) p + a)            (6) S_p <= 1 / (1 - a)
  (9) S_p = S_p1 S_p2 (TLP)                (10) E_p = S_p / (p1 p2)
  (11) beta* = beta / (beta + (1 - beta)/p2)
  (12) p2' = (1 + PRI) p2
  (13) S_p2 = 1 / (beta + (1 - beta) / (p2 (1 + PRI)))
  (14) 1 + (p - p1)/((1 - beta*) p1) = (1 + PRI*) p2
  (15) PRI* = beta/(1 - beta) (p2 - 1)
Lines: P:223-234 (1-2), P:270-290 (3-6), P:418-426 (9-10), P:493-496 (11),
P:529-538 (12), P:567-573 (13), P:578-592 (14-15).
"""
from __future__ import annotations

import math


def speedup(T1, Tp):                                   # Eq. 1
    return T1 / Tp


def efficiency(S, p):                                  # Eq. 2
    return S / p


def time_parallel(T1, p, alpha):                       # Eq. 3
    return ((1.0 - alpha) + alpha / p) * T1


def amdahl_speedup(p, alpha):                          # Eq. 4
    return p / (p - alpha * (p - 1))


def amdahl_efficiency(p, alpha):                       # Eq. 5
    return 1.0 / ((1.0 - alpha) * p + alpha)


def amdahl_limit(alpha):                               # Eq. 6
    return math.inf if alpha >= 1.0 else 1.0 / (1.0 - alpha)


def tlp_speedup(p1, a1, p2, a2):                       # Eq. 9
    return amdahl_speedup(p1, a1) * amdahl_speedup(p2, a2)


def tlp_efficiency(p1, a1, p2, a2):                    # Eq. 10
    return tlp_speedup(p1, a1, p2, a2) / (p1 * p2)


def beta_star(beta, p2):                               # Eq. 11
    return beta / (beta + (1.0 - beta) / p2)


def p2_actual(p2, pri):                                # Eq. 12
    return (1.0 + pri) * p2


def tlpdpr_speedup2(beta, p2, pri):                    # Eq. 13
    return 1.0 / (beta + (1.0 - beta) / (p2 * (1.0 + pri)))


def pri_condition_residual(p, p1, p2, beta, pri):      # Eq. 14 (zero at PRI*)
    return 1.0 + (p - p1) / ((1.0 - beta_star(beta, p2)) * p1) - (1.0 + pri) * p2


def pri_star(beta, p2):                                # Eq. 15
    return beta / (1.0 - beta) * (p2 - 1)


def fit_alpha(ps, speedups):
    """Least-squares alpha of Eq. 4 for measured (p, S_p) pairs (1-D search on [0, 1])."""
    def err(a):
        return sum((amdahl_speedup(p, a) - s) ** 2 for p, s in zip(ps, speedups))
    lo, hi = 0.0, 1.0
    for _ in range(200):                               # golden-section search
        m1 = lo + (hi - lo) * 0.381966
        m2 = hi - (hi - lo) * 0.381966
        if err(m1) < err(m2):
            hi = m2
        else:
            lo = m1
    return 0.5 * (lo + hi)


def batching_model(ms_per_step):
    """The c4 batching sweep in the paper's first-level (PSIR) terms: running n
    runs as one batch against n runs one after another on the same GPU,
    S_n = n T(1) / T(n) (Eq. 1 with T_1 = n T(1)), E_n = S_n / n (Eq. 2), and the
    alpha of Eq. 4 that fits S_n -- the share of a lone run's step that batching
    overlaps (the GPU idles that share when it holds one 2.6M-particle run)."""
    ns = sorted(ms_per_step)
    t1 = ms_per_step[ns[0]] / ns[0] if ns[0] != 1 else ms_per_step[1]
    rows = []
    for n in ns:
        S = speedup(n * t1, ms_per_step[n])
        rows.append(dict(n=n, ms=ms_per_step[n], S=S, E=efficiency(S, n)))
    alpha = fit_alpha([r["n"] for r in rows], [r["S"] for r in rows])
    return rows, alpha


if __name__ == "__main__":
    import sys
    # profiles/r01b_c4_sweep.md (ms/step per n), measured on one B200
    sweep = {1: 0.131, 4: 0.391, 16: 1.405, 64: 5.469, 256: 21.775}
    if len(sys.argv) > 1:
        sweep = {}
        for line in open(sys.argv[1]):
            parts = [p.strip() for p in line.split("|")]
            if len(parts) > 4 and parts[1].isdigit():
                sweep[int(parts[1])] = float(parts[3])
    rows, alpha = batching_model(sweep)
    print("| n | ms/step | S_n (Eq. 1) | E_n (Eq. 2) | Eq. 4 at fitted alpha |")
    print("|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['n']} | {r['ms']:.3f} | {r['S']:.3f} | {r['E']:.4f} | {amdahl_speedup(r['n'], alpha):.3f} |")
    print(f"\nfitted alpha = {alpha:.4f}; Amdahl limit 1/(1-alpha) = {amdahl_limit(alpha):.3f} (Eq. 6)")
