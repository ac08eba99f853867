import dataclasses, sys, os, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import workload as W, bench
for name, cfg in (("ragged", W.CONFIGS[5]), ("uniform", dataclasses.replace(W.CONFIGS[5], k=(256, 256), q=(64, 64))),
                  ("ragged_sorted", None)):
    if cfg is None:
        # same ragged instances, reordered by size within each group (perm applied to the batch)
        cfg = W.CONFIGS[5]
        bd = W.make_batch(cfg, device="cuda")
        k = (bd.run_off[1:] - bd.run_off[:-1]) + (bd.q_off[1:] - bd.q_off[:-1])
        g = bd.dist_of.long()
        order = torch.argsort(g * 100000 + (1000 - k).long())  # group-major, big first
        ids = bd.inst_ids[order]
        bd = W.make_batch(cfg, ids.cpu(), device="cuda")
    else:
        bd = W.make_batch(cfg, device="cuda")
    s = bench.scheduler_for(cfg, bd, 0, 1, 0, 500, 0x5EED)
    co, cl = W.make_completions(cfg, 1, bd.row_ids)
    s.update_history(co, cl)
    n = bd.n
    adm = torch.empty(n, dtype=torch.int32, device="cuda"); pk = torch.empty_like(adm)
    for t in range(3):
        s.admit(bd.run_off, bd.input_len, bd.generated, bd.q_off, bd.q_input_len, bd.max_new, bd.capacity, t, admitted_out=adm, peak_out=pk)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in range(20):
        s.admit(bd.run_off, bd.input_len, bd.generated, bd.q_off, bd.q_input_len, bd.max_new, bd.capacity, t, admitted_out=adm, peak_out=pk)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(name, "ms", round(ms, 4), "slots", bd.slots(), "ns/slot", round(ms * 1e6 / bd.slots(), 4), flush=True)
    s.close(); del bd; torch.cuda.empty_cache()
