"""admit_group_kernel vs admit_kernel (PFSCHED_GROUP_KERNEL=0) vs the oracle on a scaled config 5,
per output, and for mismatching instances the exact M*(p*) recomputed from the GPU predictions.
usage (GPU box): python tools/group_kernel_check.py [N_INSTANCES]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workload as W  # noqa: E402
from harness import gpu_admit, make_oracle, make_scheduler, oracle_admit  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
cfg = W.scaled(W.CONFIGS[5], n)
b = W.make_batch(cfg)
bd = b.to("cuda")
orc = make_oracle(b)
os.environ["PFSCHED_GROUP_KERNEL"] = "1"
s1 = make_scheduler(bd, mode=0, bp=500, seed=16, R=1)
os.environ["PFSCHED_GROUP_KERNEL"] = "0"
s0 = make_scheduler(bd, mode=0, bp=500, seed=16, R=1)
g1 = gpu_admit(s1, bd, 0)
g0 = gpu_admit(s0, bd, 0)
o = oracle_admit(orc, b, mode=0, bp=500, seed=16, R=1, tick=0)
ro, qo = b.run_off.numpy(), b.q_off.numpy()
for key in ("admitted", "peak", "peak_running", "pred_run", "pred_q"):
    a1, a0, ao = (np.asarray(x[key]) for x in (g1, g0, o))
    print(key, "new!=orc", int((a1 != ao).sum()), "old!=orc", int((a0 != ao).sum()))
bad = np.nonzero(np.asarray(g1["peak"]) != np.asarray(o["peak"]))[0]
for i in bad[:6]:
    k = ro[i + 1] - ro[i]
    q = qo[i + 1] - qo[i]
    print(f"inst {i}: k={k} q={q} cap={int(b.capacity[i])} p*: new {g1['admitted'][i]} old {g0['admitted'][i]} "
          f"orc {o['admitted'][i]}  peak new {g1['peak'][i]} old {g0['peak'][i]} orc {o['peak'][i]}  "
          f"M0 new {g1['peak_running'][i]} orc {o['peak_running'][i]}")

def T_of(i, p, tau, pr, pq):
    r0, r1, q0 = ro[i], ro[i + 1], qo[i]
    lp = b.input_len.numpy()[r0:r1].astype(np.int64)
    lt = b.generated.numpy()[r0:r1].astype(np.int64)
    r = pr[r0:r1].astype(np.int64) - lt
    a = lp + lt
    qlp = b.q_input_len.numpy()[q0:q0 + p].astype(np.int64)
    qr = pq[q0:q0 + p].astype(np.int64)
    rr = np.concatenate([r, qr]); aa = np.concatenate([a, qlp])
    m = rr >= tau
    return int((aa[m] + tau).sum())

def Mstar(i, p, pr, pq):
    r0, r1, q0 = ro[i], ro[i + 1], qo[i]
    lt = b.generated.numpy()[r0:r1].astype(np.int64)
    taus = set((pr[r0:r1].astype(np.int64) - lt).tolist()) | set(pq[q0:q0 + p].astype(np.int64).tolist())
    return max(T_of(i, p, t, pr, pq) for t in taus)

pr1, pq1 = np.asarray(g1["pred_run"]), np.asarray(g1["pred_q"])
for i in bad[:3]:
    p = int(o["admitted"][i])
    print("inst", i, "M*(p*) from preds:", Mstar(i, p, pr1, pq1), "T_p(88)", T_of(i, p, 88, pr1, pq1),
          "T_p(87)", T_of(i, p, 87, pr1, pq1), "T_R(88)", T_of(i, 0, 88, pr1, pq1))
