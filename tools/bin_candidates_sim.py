"""Numpy simulation of the sort-free bin-edge evaluation: how many bins need
exact refinement per M* evaluation. Usage: PYTHONPATH=. python tools/bin_candidates_sim.py CFG N NBINS"""
import numpy as np, torch, workload as W, sys
sys.path.insert(0,'tests')
from harness import make_oracle, oracle_admit, np32
cfg = W.scaled(W.CONFIGS[int(sys.argv[1])], int(sys.argv[2]))
NB=int(sys.argv[3]); 
b = W.make_batch(cfg); orc = make_oracle(b)
o = oracle_admit(orc, b, mode=0, bp=500, seed=7, R=1, tick=0)
ro, qo = np32(b.run_off), np32(b.q_off)
lt, lp, qlp = np32(b.generated), np32(b.input_len), np32(b.q_input_len)
Lmax = cfg.max_len
KO = int(sys.argv[4]) if len(sys.argv) > 4 else 5   # 2^KO sub-bins per octave
E = 1 << (KO + 1)                                    # exact bins for r <= E
def f_of(r, s):
    r0 = 1 << (s + KO)
    if r <= E: return r-1
    if r < r0:
        o = int(np.floor(np.log2(r))); return E + (1<<KO)*(o-KO-1) + ((r - (1<<o)) >> (o-KO))
    return E + (1<<KO)*(s-1) + ((r-r0)>>s)
s=1
while s < 30 and f_of(Lmax, s) > NB-1: s+=1
while f_of(Lmax, s) > NB-1: s+=1
fmap = np.array([0]+[f_of(r,s) for r in range(1,Lmax+1)])
lo_edge = np.zeros(NB, int); hi_edge=np.zeros(NB,int)
for f in range(NB):
    rs = np.nonzero(fmap[1:]==f)[0]+1
    if len(rs): lo_edge[f]=rs.min(); hi_edge[f]=rs.max()
    else: lo_edge[f]=hi_edge[f]=10**9
ncand=[]; work=[]
for i in range(b.n):
    for which in ('R','all'):
        r = o['pred_run'][ro[i]:ro[i+1]]-lt[ro[i]:ro[i+1]]; a = lp[ro[i]:ro[i+1]]+lt[ro[i]:ro[i+1]]
        if which=='all':
            r = np.concatenate([r, o['pred_q'][qo[i]:qo[i+1]]]); a = np.concatenate([a, qlp[qo[i]:qo[i+1]]])
        f = fmap[r]
        # bins in descending r order = descending f
        SA = np.bincount(f, weights=a, minlength=NB)[::-1]; SN = np.bincount(f, minlength=NB)[::-1]
        A = np.cumsum(SA); N = np.cumsum(SN)
        lo = lo_edge[::-1]; hi = hi_edge[::-1]
        valid = lo < 10**9
        LB = np.where(valid, A + lo*N, 0); UB = np.where(valid, A + hi*N, 0)
        exact = (hi==lo) | (SN==0) 
        L = max(LB.max(), np.where(exact & valid, UB, 0).max())
        cand = (~exact) & valid & (UB > L)
        ncand.append(cand.sum()); work.append((SN[cand]**2).sum())
print('NB',NB,'KO',KO,'s',s,'mean candidates', np.mean(ncand), 'max', np.max(ncand), 'mean pair work', np.mean(work), 'p90', np.percentile(work,90))
