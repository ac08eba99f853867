"""Numpy simulation of the cutting-plane admission search: counts how many
(p_max, probe) iterations it needs per instance and asserts the result equals the
oracle p*. Usage: PYTHONPATH=. python tools/cutting_plane_sim.py CONFIG INSTANCES"""
import numpy as np, torch, workload as W, oracle as O, sys
sys.path.insert(0,'tests')
from harness import make_oracle, oracle_admit, np32
cfg = W.scaled(W.CONFIGS[int(sys.argv[1])], int(sys.argv[2]))
b = W.make_batch(cfg)
orc = make_oracle(b)
o = oracle_admit(orc, b, mode=0, bp=500, seed=7, R=1, tick=0)
ro, qo = np32(b.run_off), np32(b.q_off)
lp, lt, qlp, cap = np32(b.input_len), np32(b.generated), np32(b.q_input_len), np32(b.capacity)
pr, pq = o['pred_run'], o['pred_q']
iters=[]; lens=[]
for i in range(b.n):
    a = np.concatenate([lp[ro[i]:ro[i+1]]+lt[ro[i]:ro[i+1]], qlp[qo[i]:qo[i+1]]]).astype(np.int64)
    r = np.concatenate([pr[ro[i]:ro[i+1]]-lt[ro[i]:ro[i+1]], pq[qo[i]:qo[i+1]]]).astype(np.int64)
    k = ro[i+1]-ro[i]; q = qo[i+1]-qo[i]
    j = np.concatenate([np.zeros(k,np.int64), np.arange(1,q+1)])
    order = np.argsort(-r, kind='stable'); a,r,j = a[order],r[order],j[order]
    C = (10000-500)*int(cap[i])
    def V(p):
        inc = (j<=p)
        A = np.cumsum(a*inc); N = np.cumsum(inc)
        return A + r*N
    fits = lambda m: m*10000 <= C
    v0 = V(0); vq = V(q)
    if not fits(v0.max()): iters.append(0); continue
    if fits(vq.max()): iters.append(0); continue
    ph = q; it=0
    while True:
        v = V(ph); m = v.max()
        if fits(m): break
        it+=1
        t = int(np.argmax(v))  # most violating position
        # p_max at position t: prefix over queue in FIFO order of entries at sorted pos <= t
        w = np.zeros(q+1, np.int64)
        for pos in range(t+1):
            if j[pos]>0: w[j[pos]] = a[pos] + r[t]
        cs = np.cumsum(w)
        base = v0[t]
        ok = np.nonzero((base + cs)*10000 <= C)[0]
        ph = int(ok.max())
    iters.append(it)
    assert ph == o['admitted'][i], (i, ph, o['admitted'][i])
it = np.array(iters); print('instances', b.n, 'iters hist', np.bincount(it), 'mean', it.mean())
