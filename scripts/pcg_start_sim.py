"""PCG iterations per Algorithm-2 step for different PCG starts (dense numpy, small
BA / RGG graphs): plain X^k, rho extrapolation (R23), Galerkin over the last m step
differences (R27, "gal"), plus the previous solve's Krylov directions ("galk"),
across columns ("...x"), or exact low eigenvectors ("eig").  Design study for R27;
usage: python scripts/pcg_start_sim.py 1500 ba "rho:0,gal:2,gal:8" """
import sys, numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from workloads import graphs
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import shortest_path

n0 = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
kind = sys.argv[2] if len(sys.argv) > 2 else 'ba'
dim = 2
if kind == 'ba':
    g = graphs.barabasi_albert(n0, 3, 7)
elif kind == 'rgg':
    g = graphs.random_geometric_graph(n0, 6, 7); dim = 3
else:
    g = graphs.gnm_graph(n0, 2 * n0, 7)
n = g.n
H = shortest_path(csr_matrix((np.ones(len(g.col)), g.col, g.row_ptr), shape=(g.n, g.n)), unweighted=True)
k = np.sqrt(1.0 / n)
D = k * H
W = np.zeros_like(D); off = H > 0; W[off] = D[off] ** -2
L = np.diag(W.sum(1)) - W
dg = np.diag(L).copy()

def stress(X):
    r = np.sqrt(((X[:, None, :] - X[None, :, :]) ** 2).sum(-1))
    iu = np.triu_indices(n, 1)
    return float((W[iu] * (r[iu] - D[iu]) ** 2).sum())

def RX(X):
    diff = X[:, None, :] - X[None, :, :]
    r = np.sqrt((diff ** 2).sum(-1))
    c = np.zeros_like(r); m = (r > 0) & off
    c[m] = W[m] * D[m] / r[m]
    return (c[:, :, None] * diff).sum(1)

RT = float(__import__("os").environ.get("RT", "1e-6"))
def pcg(b, x0, rtol=None):
    rtol = rtol or RT
    x = x0.copy(); r = b - L @ x; its = 0
    bb = (b * b).sum(0)
    act = (r * r).sum(0) > rtol ** 2 * bb
    z = r / dg[:, None]; p = z.copy(); rz = (r * z).sum(0)
    P, AP = [], []
    while act.any():
        Ap = L @ p; its += 1
        P.append(p.copy()); AP.append(Ap.copy())
        a = np.where(act, rz / (p * Ap).sum(0), 0.0)
        x += a * p; r -= a * Ap
        z = r / dg[:, None]; rzn = (r * z).sum(0)
        act = act & ((r * r).sum(0) > rtol ** 2 * bb)
        p = z + (rzn / rz) * p; rz = rzn
        if its > 500: break
    return x, its, P, AP

EV=None
def run(strategy, m=4, omega=1.5, tol=1e-4, maxit=500, seed=5):
    X = graphs.init_positions(n, dim, seed)
    f = stress(X); hist = []; Vs = []; AVs = []; Xprev = None; rho = 0.0
    A = L @ X
    its_tot = []; Pk = []; APk = []
    for it in range(maxit):
        b = RX(X)
        if strategy == 'plain' or Xprev is None:
            x0 = X.copy()
        elif strategy == 'rho':
            x0 = X + rho * (X - Xprev)
        else:  # galerkin over last m differences, per column
            x0 = X.copy()
            r = b - A
            if Vs:
                for c in range(dim):
                    cols = range(dim) if strategy.endswith('x') else [c]
                    if strategy.startswith('eig'):
                        V = np.concatenate([EV, np.stack([v[:, c] for v in Vs[-4:]], 1)], 1); AV = L @ V
                    else:
                      V = np.stack([v[:, cc] for v in Vs[-m:] for cc in cols] + [q[:, cc] for q in Pk for cc in cols], 1)
                      AV = np.stack([a[:, cc] for a in AVs[-m:] for cc in cols] + [q[:, cc] for q in APk for cc in cols], 1)
                    G = V.T @ AV; G = 0.5 * (G + G.T)
                    rhs = V.T @ r[:, c]
                    w_, U = np.linalg.eigh(G)
                    keep = w_ > 1e-12 * w_.max()
                    y = U[:, keep] @ ((U[:, keep].T @ rhs) / w_[keep])
                    x0[:, c] += V @ y
        xn, its, P_, AP_ = pcg(b, x0)
        if 'k' in strategy: Pk, APk = P_, AP_
        its_tot.append(its)
        fn = stress(xn)
        Xt = (1 + omega) * xn - omega * X
        ft = stress(Xt)
        if ft <= fn:
            Xnew, fnew = Xt, ft
        else:
            Xnew, fnew = xn, fn
        # rho from this step (as the GPU: <Xn - Xk, Xk - Xprev> / |Xk - Xprev|^2)
        if Xprev is not None:
            dp = X - Xprev; rho = float(((xn - X) * dp).sum() / (dp * dp).sum())
        Anew = L @ Xnew
        Vs.append(Xnew - X); AVs.append(Anew - A)
        Xprev, X, A = X, Xnew, Anew
        rel = (f - fnew) / f
        f = fnew
        if rel < tol: break
    return it + 1, f, its_tot

def eig_basis(m):
    global EV
    w_, U = np.linalg.eigh(L)
    EV = U[:, 1:m + 1]
for strat, m in [(a, int(b)) for a, b in (t.split(':') for t in sys.argv[3].split(','))]:
    if strat.startswith('eig'): eig_basis(m)
    iters, f, its = run(strat, m)
    its = np.array(its)
    print(f"{kind} n={n} {strat:5s} m={m}: steps {iters} f {f:.6e} pcg/step mean {its.mean():.2f} "
          f"(after 10: {its[10:].mean() if len(its) > 10 else float('nan'):.2f}) total {its.sum()}", flush=True)
