"""NumPy prototype of the warp-partitioned ALS solver (k_als.cu), lane by lane, to check the
index bookkeeping against the oracle's als_baseline before the CUDA version.  Not shipped code.

Segments s = 0..P-1 (lane s), rows [b_s, e_s).  Separators: the last two rows of every segment
but the last.  Interior rows are eliminated by an LDL^T in direction dir (alternating per
iteration); the Schur complement on the separators (2x2-block tridiagonal) is solved by parallel
cyclic reduction; pass B forward-substitutes the corrected right-hand side; the next iteration's
pass A back-substitutes it (fused with the next factorisation)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import fkk_oracle as O  # noqa: E402


def d0(i, M):
    return 1.0 if i in (0, M - 1) else (5.0 if i in (1, M - 2) else 6.0)


def d1(i, M):  # coupling (i, i+1)
    return -2.0 if i in (0, M - 2) else -4.0


def als_part(y, lam=1e4, p=1e-3, iters=10, P=32):
    M = len(y)
    P = min(P, M // 4)
    b = [(s * M) // P for s in range(P + 1)]
    q = 1.0 - p
    nseg = P
    # per-lane state
    n = [(b[s + 1] - b[s]) - (2 if s < P - 1 else 0) for s in range(P)]
    l1 = [np.zeros(n[s]) for s in range(P)]
    rD = [np.zeros(n[s]) for s in range(P)]
    G = [np.zeros(n[s]) for s in range(P)]
    w = np.ones(M)
    xsep = np.zeros((P, 2))   # lane s: separator S_s rows (e-2, e-1)
    out = np.zeros(M)

    def rows_in_order(s, dr):
        r = np.arange(b[s], b[s] + n[s])
        return r if dr == 0 else r[::-1]

    def coupling(i, j):  # A[i, j] off-diagonal band value (|i-j| in {1,2})
        lo = min(i, j)
        return lam * d1(lo, M) if abs(i - j) == 1 else lam

    for it in range(iters + 1):
        dr = it & 1
        C = np.zeros((P, 4, 4))
        Cf = np.zeros((P, 4))
        for s in range(P):
            rows = rows_in_order(s, dr)
            nn = n[s]
            # previous system back-substitution (reverse of its elimination order = this order)
            if it > 0:
                z1 = z2 = 0.0
                for t in range(nn):
                    tt = nn - 1 - t          # index in the previous elimination order
                    i = rows[t]
                    l2 = lam * rD[s][tt + 2] if False else None  # placeholder (not used)
                    # previous order: position tt; its l1/l2 couple to tt+1, tt+2 (already done: z1, z2)
                    l1p = l1[s][tt] if tt + 1 < nn else 0.0
                    l2p = lam * rD[s][tt] if tt + 2 < nn else 0.0
                    zv = G[s][tt] - l1p * z1 - l2p * z2
                    z2, z1 = z1, zv
                    out[i] = zv
                    w[i] = p if y[i] > zv else q
            if it == iters:
                continue
            # canonical spike columns [L0, L1, R0, R1] = rows [b-2, b-1, e-2, e-1]
            e = b[s + 1]
            hasL, hasR = s > 0, s < P - 1
            cols = [b[s] - 2, b[s] - 1, e - 2, e - 1]
            if dr == 0:
                na, nf, fa, ff = 1, 0, 2, 3
                hasN, hasF = hasL, hasR
            else:
                na, nf, fa, ff = 2, 3, 1, 0
                hasN, hasF = hasR, hasL
            Dm1 = Dm2 = 0.0
            L1m1 = 0.0
            rDm1 = rDm2 = 0.0
            gf1 = gf2 = 0.0
            ga1 = ga2 = gb1 = gb2 = 0.0   # near columns na (a), nf (b)
            Yst = []
            new_l1 = np.zeros(nn)
            new_rD = np.zeros(nn)
            for t in range(nn):
                i = rows[t]
                a0 = w[i] + lam * d0(i, M)
                a1 = coupling(i, rows[t + 1]) if t + 1 < nn else 0.0
                D = a0 - L1m1 * L1m1 * Dm1 - lam * lam * rDm2
                rd = 1.0 / D
                l1n = (a1 - lam * L1m1 * (1.0 if t >= 1 else 0.0)) * rd if t + 1 < nn else 0.0
                # careful: the L2m1*L1m1*Dm1 term = lam * L1m1 only when row t-1 has an l2 to t+1
                L2m2 = lam * rDm2
                f = w[i] * y[i]
                gf = f - L1m1 * gf1 - L2m2 * gf2
                ea = (coupling(i, cols[na]) if (hasN and abs(i - cols[na]) <= 2) else 0.0)
                eb = (coupling(i, cols[nf]) if (hasN and abs(i - cols[nf]) <= 2) else 0.0)
                ga = ea - L1m1 * ga1 - L2m2 * ga2
                gb = eb - L1m1 * gb1 - L2m2 * gb2
                C[s, na, na] += ga * ga * rd
                C[s, na, nf] += ga * gb * rd
                C[s, nf, nf] += gb * gb * rd
                Cf[s, na] += ga * gf * rd
                Cf[s, nf] += gb * gf * rd
                Yst.append((ga, gb, gf, rd))
                new_l1[t] = l1n
                new_rD[t] = rd
                Dm2, Dm1 = Dm1, D
                rDm2, rDm1 = rDm1, rd
                L1m1 = l1n
                gf2, gf1 = gf1, gf
                ga2, ga1 = ga1, ga
                gb2, gb1 = gb1, gb
            C[s, nf, na] = C[s, na, nf]
            l1[s], rD[s] = new_l1, new_rD
            # far columns at t = nn-2, nn-1
            if hasF:
                Yfa = np.zeros(nn)
                Yff = np.zeros(nn)
                for t in (nn - 2, nn - 1):
                    i = rows[t]
                    efa = coupling(i, cols[fa]) if abs(i - cols[fa]) <= 2 else 0.0
                    eff = coupling(i, cols[ff]) if abs(i - cols[ff]) <= 2 else 0.0
                    pa = Yfa[t - 1] if t >= 1 else 0.0
                    pb = Yff[t - 1] if t >= 1 else 0.0
                    Yfa[t] = efa - (new_l1[t - 1] if t >= 1 else 0.0) * pa
                    Yff[t] = eff - (new_l1[t - 1] if t >= 1 else 0.0) * pb
                for t in (nn - 2, nn - 1):
                    ga, gb, gf, rd = Yst[t]
                    yy = {na: ga, nf: gb, fa: Yfa[t], ff: Yff[t]}
                    for x in (fa, ff):
                        for z in (na, nf, fa, ff):
                            if z in (na, nf):
                                C[s, x, z] += yy[x] * yy[z] * rd
                                C[s, z, x] += yy[x] * yy[z] * rd
                            elif z >= x or True:
                                pass
                    C[s, fa, fa] += Yfa[t] * Yfa[t] * rd
                    C[s, fa, ff] += Yfa[t] * Yff[t] * rd
                    C[s, ff, fa] += Yfa[t] * Yff[t] * rd
                    C[s, ff, ff] += Yff[t] * Yff[t] * rd
                    Cf[s, fa] += Yfa[t] * gf * rd
                    Cf[s, ff] += Yff[t] * gf * rd
        if it == iters:
            break
        # reduced system on separators s = 0..P-2 (rows e_s-2, e_s-1)
        ns = P - 1
        Dm = np.zeros((ns, 2, 2))
        Um = np.zeros((ns, 2, 2))
        r = np.zeros((ns, 2))
        for s in range(ns):
            e = b[s + 1]
            i0, i1 = e - 2, e - 1
            Dm[s] = [[w[i0] + lam * d0(i0, M), lam * d1(i0, M)], [lam * d1(i0, M), w[i1] + lam * d0(i1, M)]]
            Dm[s] -= C[s][2:, 2:] + C[s + 1][:2, :2]
            Um[s] = -C[s + 1][:2, 2:]
            r[s] = [w[i0] * y[i0], w[i1] * y[i1]]
            r[s] -= Cf[s][2:] + Cf[s + 1][:2]
        # PCR
        Lm = np.zeros((32, 2, 2)); Dd = np.tile(np.eye(2), (32, 1, 1)); Uu = np.zeros((32, 2, 2)); rr = np.zeros((32, 2))
        Dd[:ns] = Dm; Uu[:ns] = Um; rr[:ns] = r
        for s in range(1, ns):
            Lm[s] = Um[s - 1].T
        h = 1
        while h < 32:
            Pm = np.array([np.linalg.solve(Dd[j], Lm[j]) for j in range(32)])
            Qm = np.array([np.linalg.solve(Dd[j], Uu[j]) for j in range(32)])
            sm = np.array([np.linalg.solve(Dd[j], rr[j]) for j in range(32)])
            nL = np.zeros_like(Lm); nU = np.zeros_like(Uu); nD = Dd.copy(); nr = rr.copy()
            for i in range(32):
                if i - h >= 0:
                    nL[i] = -Lm[i] @ Pm[i - h]
                    nD[i] -= Lm[i] @ Qm[i - h]
                    nr[i] -= Lm[i] @ sm[i - h]
                if i + h < 32:
                    nU[i] = -Uu[i] @ Qm[i + h]
                    nD[i] -= Uu[i] @ Pm[i + h]
                    nr[i] -= Uu[i] @ sm[i + h]
            Lm, Uu, Dd, rr = nL, nU, nD, nr
            h *= 2
        x = np.array([np.linalg.solve(Dd[s], rr[s]) for s in range(32)])
        xsep[:ns] = x[:ns]
        for s in range(ns):
            e = b[s + 1]
            out[e - 2], out[e - 1] = x[s]
        # pass B: corrected RHS forward substitution
        for s in range(P):
            rows = rows_in_order(s, dr)
            nn = n[s]
            e = b[s + 1]
            xs = {b[s] - 2: xsep[s - 1][0] if s > 0 else 0.0, b[s] - 1: xsep[s - 1][1] if s > 0 else 0.0,
                  e - 2: xsep[s][0] if s < P - 1 else 0.0, e - 1: xsep[s][1] if s < P - 1 else 0.0}
            g1 = g2 = 0.0
            for t in range(nn):
                i = rows[t]
                f = w[i] * y[i]
                for j, xv in xs.items():
                    if (j < b[s] or j >= b[s] + nn) and abs(i - j) <= 2 and 0 <= j < M:
                        f -= coupling(i, j) * xv
                L1m1 = l1[s][t - 1] if t >= 1 else 0.0
                L2m2 = lam * rD[s][t - 2] if t >= 2 else 0.0
                g = f - L1m1 * g1 - L2m2 * g2
                G[s][t] = g * rD[s][t]
                g2, g1 = g1, g
        # separator weights for the next iteration
        for s in range(ns):
            e = b[s + 1]
            for i in (e - 2, e - 1):
                w[i] = p if y[i] > out[i] else q
    return out


if __name__ == "__main__":
    rng = np.random.default_rng(0)
    for M in (64, 100, 512, 1000):
        x = np.linspace(0, 1, M)
        y = np.sin(7 * x) + 0.3 * x + 0.05 * rng.standard_normal(M) + (np.abs(x - 0.4) < 0.02) * 2.0
        ref = O.als_baseline(y, O.Params())[0]
        got = als_part(y)
        print(M, np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
