"""Design study: PCG iterations of Jacobi vs an additive two-level
preconditioner M^-1 = D^-1 + Z (Z^T L Z)^-1 Z^T (Z = greedy BFS aggregates of `agg`
vertices) on the dense L^W of a small graph, from a warm start, to 1e-6 and 1e-9.
usage: python scripts/twolevel_sim.py rgg|ba N AGG"""
import sys, numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from workloads import graphs
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import shortest_path, breadth_first_order
kind=sys.argv[1]; n0=int(sys.argv[2]); agg=int(sys.argv[3])
if kind=='rgg': g=graphs.random_geometric_graph(n0,6,7); dim=3
else: g=graphs.barabasi_albert(n0,3,7); dim=2
n=g.n
A=csr_matrix((np.ones(len(g.col)), g.col, g.row_ptr), shape=(n,n))
H=shortest_path(A, unweighted=True)
W=np.zeros_like(H); off=H>0; W[off]=H[off]**-2
L=np.diag(W.sum(1))-W; dg=np.diag(L).copy()
# aggregates: greedy BFS balls of size agg
lab=-np.ones(n,int); c=0
order=np.argsort(-np.asarray(A.sum(1)).ravel()) if kind=='ba' else np.arange(n)
for s in range(n):
    if lab[s]>=0: continue
    # grow from s by BFS over unlabeled
    q=[s]; lab[s]=c; cnt=1; qi=0
    while qi<len(q) and cnt<agg:
        u=q[qi]; qi+=1
        for v in g.col[g.row_ptr[u]:g.row_ptr[u+1]]:
            if lab[v]<0 and cnt<agg:
                lab[v]=c; q.append(v); cnt+=1
    c+=1
nc=c
Z=np.zeros((n,nc)); Z[np.arange(n),lab]=1
Ac=Z.T@L@Z + (dg.mean()/n)*np.ones((nc,nc))  # regularise the constant mode
Aci=np.linalg.inv(Ac)
rng=np.random.default_rng(1)
X=rng.random((n,dim))
b=L@(X+0.01*rng.standard_normal((n,dim)))   # a consistent rhs near X
b-=b.mean(0)
def pcg(prec, x0, rtol):
    x=x0.copy(); r=b-L@x; bb=np.linalg.norm(b)
    z=prec(r); p=z.copy(); rz=(r*z).sum(); its=0
    while np.linalg.norm(r)>rtol*bb and its<2000:
        Ap=L@p; a=rz/(p*Ap).sum(); x+=a*p; r-=a*Ap; z=prec(r); rzn=(r*z).sum(); p=z+rzn/rz*p; rz=rzn; its+=1
    return its
jac=lambda r: r/dg[:,None]
two=lambda r: r/dg[:,None] + Z@(Aci@(Z.T@r))
for rt in (1e-6,1e-9):
    print(kind, n, 'agg',agg,'nc',nc,'rtol',rt,'jacobi',pcg(jac,X,rt),'two-level',pcg(two,X,rt))
