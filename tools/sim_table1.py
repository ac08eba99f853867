"""Table 1 re-run on the GPU simulator (pf_sim_*, NEXT-2).

Synthetic Distribution-1/2/3 request lists at the paper's scale: a KV
pool of 16 worst-case requests (16 × 8192 = 131,072 tokens for D1/D3, about the KV
capacity of Llama-2-7B on an A100-80G), w = 1000 with a steady-state window, every
request queued at t = 0. Columns as the paper: decoding steps (mean per instance),
current consumed memory, future required memory (means over iterations, % of M) and
evicted requests (% of requests). Absolute values are not comparable with the paper
(no model timings, synthetic lengths); the ordering of the rows is the claim.

Usage: python tools/sim_table1.py [--inst 16] [--req 400] [--out profiles/r01/sim_table1.txt]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2507_10150_b200 as P  # noqa: E402
import workload.sim as S  # noqa: E402
from workload.gen import D1, D2, D3  # noqa: E402

ROWS = {
    D1: [("Theoretical optimum", P.PF_SIM_OPTIMUM, 0), ("Past-Future (reserved=3%)", P.PF_SIM_PAST_FUTURE, 300),
         ("Past-Future (reserved=5%)", P.PF_SIM_PAST_FUTURE, 500),
         ("Past-Future (reserved=10%)", P.PF_SIM_PAST_FUTURE, 1000),
         ("Aggressive (watermark=99%)", P.PF_SIM_AGGRESSIVE, 9900),
         ("Aggressive (watermark=95%)", P.PF_SIM_AGGRESSIVE, 9500),
         ("Aggressive (watermark=90%)", P.PF_SIM_AGGRESSIVE, 9000),
         ("Conservative (no overcommit)", P.PF_SIM_CONSERVATIVE, 10000),
         ("Conservative (overcommit=150%)", P.PF_SIM_CONSERVATIVE, 15000)],
}
ROWS[D3] = ROWS[D1]
ROWS[D2] = ROWS[D1][:-1] + [("Conservative (overcommit=125%)", P.PF_SIM_CONSERVATIVE, 12500)]
NAMES = {D1: "Distribution-1 (decode-heavy)", D2: "Distribution-2 (balanced)",
         D3: "Distribution-3 (prefill-heavy)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--inst", type=int, default=16)
    ap.add_argument("--req", type=int, default=400)
    ap.add_argument("--slots", type=int, default=16)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    lines = [f"# Table 1 re-run on the GPU simulator: {a.inst} instances x {a.req} requests per "
             f"distribution, KV pool = {a.slots} worst-case requests, w = 1000, sampling mode, R = 1",
             f"{'Dataset':32s} {'Method':32s} {'Decoding Steps':>15s} {'Consumed':>9s} {'Future':>9s} "
             f"{'Evicted':>9s} {'iters/s':>9s}"]
    for cls in (D1, D2, D3):
        w = S.make_sim_workload(cls, a.inst, a.req, div=1, slots=a.slots, window=1000)
        d = {k: (v.cuda() if torch.is_tensor(v) else v) for k, v in w.items()}
        cap = int(w["capacity"][0])
        for name, pol, bp in ROWS[cls]:
            sim = P.Simulator(req_off=d["req_off"], req_input=d["req_input"], req_output=d["req_output"],
                              max_new=d["max_new"], capacity=d["capacity"], policy=pol, param_bp=bp,
                              window=1000, max_len=w["max_len"], max_input_len=w["max_input_len"],
                              max_entries=256, init_history=d["init_history"], seed=0x7AB1E1)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            iters = sim.run(chunk=1024)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            m = sim.metrics()[0].cpu().numpy()
            assert sim.device_error() == (0, 0)
            tot = m.sum(0)
            steps = m[:, 1].mean()
            cons = 100.0 * tot[4] / (tot[6] * cap)
            fut = 100.0 * tot[5] / (tot[6] * cap)
            ev = 100.0 * tot[2] / (a.inst * a.req)
            lines.append(f"{NAMES[cls]:32s} {name:32s} {steps:15.0f} {cons:8.2f}% {fut:8.2f}% {ev:8.2f}% "
                         f"{iters / dt:9.0f}")
            print(lines[-1], flush=True)
            sim.close()
    if a.out:
        with open(a.out, "w") as f:
            f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
