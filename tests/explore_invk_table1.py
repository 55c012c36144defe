# Exploration of INVK readings against Table 1 on the 16^3 two-level problem:
# K at omega = 1 and at omega_opt = 2/(lmin+lmax) of M^-1 A, for IC(0) + truncated inverse (fill 0/1),
# D = IC pivots or diag(A), positional dropping of the exact inverse, exact IC(0); and min over omega.
# Test infrastructure (imports oracle/); see DESIGN.md 8e.
import sys, numpy as np, scipy.linalg as sl, scipy.sparse as sp, scipy.sparse.linalg as sla
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
def K_pair(Minv):
    ev = np.linalg.eigvals(Minv @ Ad).real
    wopt = 2.0 / (ev.min() + ev.max())
    return K_of_Minv(Minv, 1.0), K_of_Minv(Minv, wopt), ev.min(), ev.max()
# IC(0) on the pattern of A (lower): A = L D L^T, L unit lower
pat = Ad != 0
L = np.eye(n); d = np.zeros(n)
Al = np.tril(Ad)
for i in range(n):
    for j in np.nonzero(pat[i, :i])[0]:
        s = Ad[i, j] - sum(L[i, k] * L[j, k] * d[k] for k in np.nonzero(pat[i, :j] & pat[j, :j])[0])
        L[i, j] = s / d[j]
    d[i] = Ad[i, i] - sum(L[i, k] ** 2 * d[k] for k in np.nonzero(pat[i, :i])[0])
print("IC0 pivots range", d.min(), d.max())
Linv = np.linalg.inv(L)          # exact L^{-1}
Zex = Linv.T                      # Z = L^{-T}
# level-of-fill pattern of L^{-1}: level(i,j) by symbolic powers of the strictly lower part
Ls = (np.abs(np.tril(L, -1)) > 0).astype(float)
def lev_pattern(k):
    Pm = np.eye(n) > 0; cur = np.eye(n)
    for _ in range(k + 1):
        cur = (cur @ Ls > 0).astype(float) if _ > 0 else Ls.copy()
        Pm |= cur > 0
    return Pm
def trunc_inverse(pattern_lower):
    # W ~ L^{-1} on the given lower pattern via the column recurrence W = I - (L - I) W restricted
    W = np.zeros((n, n))
    N = L - np.eye(n)
    for j in range(n):
        w = np.zeros(n); w[j] = 1.0
        for i in range(j + 1, n):
            if pattern_lower[i, j]:
                w[i] = -N[i, :i] @ w[:i]
        W[:, j] = w
    return W
for k in (0, 1):
    pl = lev_pattern(k)
    W = trunc_inverse(pl)   # W ~ L^{-1}
    Z = W.T
    print("fill", k, "pattern nnz/row %.1f" % (pl.sum() / n))
    print("  Z D^-1 Z^T (IC pivots):  K(1), K(opt), lmin, lmax =", K_pair(Z @ np.diag(1 / d) @ Z.T))
    print("  Z diag(A)^-1 Z^T:         ", K_pair(Z @ np.diag(1 / np.diag(Ad)) @ Z.T))
    # positional dropping of the EXACT inverse
    Wd = np.where(pl, Linv, 0.0)
    print("  dropped exact inverse:    ", K_pair(Wd.T @ np.diag(1 / d) @ Wd))
print("exact IC0 M = L D L^T:", K_pair(np.linalg.inv(L @ np.diag(d) @ L.T)))
print("min over omega of K:")
for nm, Minv in [("fill0", None), ("fill1", None), ("exactIC0", np.linalg.inv(L @ np.diag(d) @ L.T))]:
    if Minv is None:
        k = 0 if nm == "fill0" else 1
        W = trunc_inverse(lev_pattern(k)); Minv = W.T @ np.diag(1 / d) @ W
    best = min((K_of_Minv(Minv, w), w) for w in np.linspace(0.5, 1.6, 23))
    print(" ", nm, "min K %.4f at omega %.2f" % best)
