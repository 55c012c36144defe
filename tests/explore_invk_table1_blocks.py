# Exploration (test infrastructure, imports oracle/): Table 1 K for HINVK / l1-INVK with
# the 3-D block distribution at np = 1, 8, 64, readings I1-I5; output in profiles/r02_invk_table1_blocks.txt
import sys, numpy as np, scipy.linalg as sl, scipy.sparse.linalg as sla
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import oracle as O
from inputs import poisson7
h = O.OracleHierarchy(poisson7(16, 16, 16), smooth_prolongator=0, max_levels=2, max_coarse_size=1)
Ad = h.A(0).to_scipy().toarray(); n = Ad.shape[0]
P = h.P(0).to_scipy().toarray(); D = np.diag(np.diag(Ad))
R = np.linalg.solve(P.T @ D @ P, P.T @ D); S = sl.null_space(R); SAS = S.T @ Ad @ S
def K_of_Minv(Minv, omega=1.0):
    M = np.linalg.inv(Minv) / omega
    Mbar = M.T @ np.linalg.solve(M.T + M - Ad, M)
    return sla.eigsh(S.T @ Mbar @ S, k=1, M=SAS, which="LA", tol=1e-10)[0][0]
def blocks(np_):
    q = round(np_ ** (1 / 3)); bs = 16 // q
    i = np.arange(n); x, y, z = i % 16, (i // 16) % 16, i // 256
    return (x // bs) + q * ((y // bs) + q * (z // bs))
def ic0(B):
    pat = B != 0; L = np.eye(n); d = np.zeros(n)
    for i in range(n):
        for j in np.nonzero(pat[i, :i])[0]:
            ks = np.nonzero(pat[i, :j] & pat[j, :j])[0]
            L[i, j] = (B[i, j] - np.sum(L[i, ks] * L[j, ks] * d[ks])) / d[j]
        ks = np.nonzero(pat[i, :i])[0]
        d[i] = B[i, i] - np.sum(L[i, ks] ** 2 * d[ks])
    return L, d
def trunc_inv(L, fill):
    N = np.tril(L, -1); W = np.zeros((n, n)); lev = np.full((n, n), 99)
    for i in range(n):
        row = np.zeros(n); lv = np.full(n, 99)
        ks = np.nonzero(N[i])[0]
        lv[ks] = 0
        for k in ks:
            cols = np.nonzero(W[k])[0]
            row[cols] += N[i, k] * W[k, cols]
            lv[cols] = np.minimum(lv[cols], lev[k, cols] + 1)
        keep = lv <= fill
        W[i, keep] = -row[keep]; lev[i, keep] = lv[keep]
        W[i, i] = 1.0; lev[i, i] = 0
    return W
for np_ in (1, 8, 64):
    b = blocks(np_); same = b[:, None] == b[None, :]
    for l1 in (0, 1):
        B = Ad * same
        if l1: B = B + np.diag((np.abs(Ad) * (~same)).sum(axis=1))
        L, d = ic0(B)
        out = []
        for fill in (0, 1):
            W = trunc_inv(L, fill)
            Minv = W.T @ np.diag(1 / d) @ W
            ev = np.linalg.eigvals(Minv @ Ad).real
            out.append((round(K_of_Minv(Minv), 4), round(K_of_Minv(Minv, 2 / (ev.min() + ev.max())), 4)))
        print("np", np_, "l1" if l1 else "H ", "fill0 K(1),K(opt)", out[0], "fill1", out[1], flush=True)
