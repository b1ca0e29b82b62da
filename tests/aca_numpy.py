"""TEST-SIDE numpy restatement of the reference ACA (gca.py:182-245), used to
cross-check the native csrc/aca.cpp on many clusters."""
import numpy as np


def aca(A, epsilon, max_rank=None):
    A = np.asarray(A)
    nr, nc = A.shape
    cap = min(nr, nc) if max_rank is None else min(max_rank, nr, nc)
    dtype = np.result_type(A.dtype, np.float64)
    U, W, rows, cols = [], [], [], []
    taken = np.zeros(nr, dtype=bool)
    est2 = 0.0
    cand = 0
    while len(rows) < cap:
        if cand >= nr or taken[cand]:
            free = np.flatnonzero(~taken)
            if free.size == 0:
                break
            cand = int(free[0])
        i = cand
        r = A[i, :].astype(dtype, copy=True)
        for u, w in zip(U, W):
            r -= u[i] * w
        j = int(np.argmax(np.abs(r)))
        taken[i] = True
        if r[j] == 0.0:
            cand = nr
            continue
        w = r / r[j]
        c = A[:, j].astype(dtype, copy=True)
        for u, ww in zip(U, W):
            c -= ww[j] * u
        U.append(c); W.append(w); rows.append(i); cols.append(j)
        nu, nw = float(np.linalg.norm(c)), float(np.linalg.norm(w))
        mix = sum((np.vdot(u, c) * np.vdot(ww, w)).real for u, ww in zip(U[:-1], W[:-1]))
        est2 = max(est2 + nu * nu * nw * nw + 2.0 * mix, 0.0)
        if nu * nw <= epsilon * np.sqrt(est2):
            break
        mag = np.abs(c)
        mag[taken] = 0.0
        cand = int(np.argmax(mag))
        if mag[cand] == 0.0:
            cand = nr
    return np.array(rows, dtype=np.int64), np.array(cols, dtype=np.int64)


def operator(A, epsilon):
    """TEST-SIDE restatement of build_interpolation_operator's pivot solve
    (reference gca.py:248-282): (row pivots, V)."""
    eps = epsilon
    for _ in range(2):
        rows, cols = aca(A, eps)
        assert rows.size, "zero Green matrix"
        block = A[np.ix_(rows, cols)]
        if np.linalg.cond(block) <= 1e14:
            A_cols = A[:, cols]
            V = np.linalg.solve(block.T, A_cols.T).T
            for _ in range(2):
                R = A_cols - V @ block
                if np.max(np.abs(R)) <= 1e-15 * max(np.max(np.abs(A_cols)), 1.0):
                    break
                V = V + np.linalg.solve(block.T, R.T).T
            return rows, V
        eps *= 0.1
    raise AssertionError("singular pivot block")
