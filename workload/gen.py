"""Deterministic synthetic inputs for the Past-Future hot path (no method arithmetic here).

Recipe:

* Streams. Every (config seed, identity, field) pair owns a SplitMix64-style
  counter stream: key = mix(mix(ident·C_ID ⊕ field·C_FIELD) ⊕ seed); the i-th
  draw is mix(key + (i+1)·γ). Integer U[lo, hi] = lo + ((x >> 32)·(hi−lo+1) >> 32).
  Written with torch int64 ops (wrapping multiply, masked logical shifts), so the
  same bits come out on CPU (tests, oracle inputs) and on CUDA (bench).
* Length classes, shaped like the paper's workloads:
    chat (ShareGPT-like, log-uniform): l_p in [2^(b+2), 2^(b+3)-1], b~U{0..8};
        L in [2^b, 2^(b+1)-1], b~U{0..10}, capped at 2048; max_new = 2048
    D1 = Distribution-1 (decode-heavy): l_p~U[32,4096], L~U[2048,4096], max_new 4096
    D2 = Distribution-2 (balanced):     l_p, L ~ U[3072,5120], max_new 5120
    D3 = Distribution-3 (prefill-heavy): l_p~U[2048,4096], L~U[32,4096], max_new 4096
    mixed: class = group mod 4 over {chat, D1, D2, D3} (the concatenated workload)
* Per instance: history = w draws of L (steady state, oldest first); running slot:
  (l_p, L), l_t ~ U[0, L-1]; queued slot: l_p; capacity = floor(cur·(10^4+f)/10^4)
  with cur = Σ_running (l_p + l_t), f ~ U{-100..2000}.
* Completions per tick: per-instance rows c ~ U{0..ceil(2k/E[L])}; shared-mode
  (group, shard) rows c ~ U{0..64}; lengths from the row's class.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional, Sequence

import torch

_M64 = (1 << 64) - 1


def _s64(c: int) -> int:
    c &= _M64
    return c - (1 << 64) if c >= (1 << 63) else c


GAMMA = _s64(0x9E3779B97F4A7C15)
_C_ID = _s64(0xD6E8FEB86659FD93)
_C_FIELD = _s64(0xA0761D6478BD642F)
_C_TICK = _s64(0xE7037ED1A0B428DB)
_M1 = _s64(0xBF58476D1CE4E5B9)
_M2 = _s64(0x94D049BB133111EB)

CHAT, D1, D2, D3, MIXED = 0, 1, 2, 3, -1
CLASS_NAMES = {CHAT: "chat", D1: "D1", D2: "D2", D3: "D3", MIXED: "mixed"}
# class -> (max_new, max_input_len, E[L] rounded)
_CLASS = {CHAT: (2048, 2047, 279), D1: (4096, 4096, 3072), D2: (5120, 5120, 4096),
          D3: (4096, 4096, 2064)}

(F_HIST_B, F_HIST, F_LP_B, F_LP, F_L_B, F_L, F_LT, F_QLP_B, F_QLP, F_QL_B, F_QL,
 F_K, F_Q, F_CAP, F_COMP_C, F_COMP_B, F_COMP, F_SHIST_B, F_SHIST) = range(1, 20)


def class_params(cls: int):
    """(max_new, max_input_len, E[L]) of a length class."""
    return _CLASS[cls]


def _lsr(x: torch.Tensor, s: int) -> torch.Tensor:
    return (x >> s) & ((1 << (64 - s)) - 1)


def _mix(z: torch.Tensor) -> torch.Tensor:
    z = z ^ _lsr(z, 30)
    z = z * _M1
    z = z ^ _lsr(z, 27)
    z = z * _M2
    z = z ^ _lsr(z, 31)
    return z


def _mix_int(z: int) -> int:
    z &= _M64
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & _M64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & _M64
    z ^= z >> 31
    return z


def _key(seed: int, ident: torch.Tensor, field: int) -> torch.Tensor:
    return _mix(_mix(ident * _C_ID ^ _s64(field * 0xA0761D6478BD642F)) ^ _s64(seed))


def _draw(key: torch.Tensor, idx: torch.Tensor) -> torch.Tensor:
    return _mix(key + (idx + 1) * GAMMA)


def _uni(x: torch.Tensor, lo, hi) -> torch.Tensor:
    return lo + _lsr(_lsr(x, 32) * (hi - lo + 1), 32)


def _lengths(cls: torch.Tensor, x1: torch.Tensor, x2: torch.Tensor, what: str) -> torch.Tensor:
    """Draw input (what='lp') or output (what='L') lengths for per-element classes."""
    if what == "lp":
        b = _uni(x1, 0, 8)
        chat_lo, chat_hi = torch.ones_like(b) << (b + 2), (torch.ones_like(b) << (b + 3)) - 1
        tab = {D1: (32, 4096), D2: (3072, 5120), D3: (2048, 4096)}
    else:
        b = _uni(x1, 0, 10)
        chat_lo, chat_hi = torch.ones_like(b) << b, (torch.ones_like(b) << (b + 1)) - 1
        tab = {D1: (2048, 4096), D2: (3072, 5120), D3: (32, 4096)}
    lo, hi = chat_lo, chat_hi
    for c, (l, h) in tab.items():
        m = cls == c
        lo = torch.where(m, torch.full_like(lo, l), lo)
        hi = torch.where(m, torch.full_like(hi, h), hi)
    v = _uni(x2, lo, hi)
    if what == "L":
        v = torch.where(cls == CHAT, v.clamp(max=2048), v)
    return v


@dataclasses.dataclass(frozen=True)
class WorkloadConfig:
    name: str
    n_instances: int
    k: tuple            # inclusive range of running requests per instance
    q: tuple            # inclusive range of queued requests per instance (0,0 = estimate only)
    window: int         # per-instance w, or global W = shards x W/shards in shared mode
    max_len: int        # Lmax: output lengths live in [1, Lmax]
    cls: int            # length class, or MIXED (class = group mod 4)
    n_groups: int = 0   # 0 = per-instance histories; G = shared group histories
    shards: int = 8
    seed: int = 0x2507101500000000

    @property
    def shared(self) -> bool:
        return self.n_groups > 0

    @property
    def max_entries(self) -> int:
        return self.k[1] + self.q[1]

    @property
    def max_input_len(self) -> int:
        if self.cls == MIXED:
            return max(v[1] for v in _CLASS.values())
        return _CLASS[self.cls][1]

    @property
    def members_per_group(self) -> int:
        return self.n_instances // self.n_groups if self.shared else 0

    @property
    def row_window(self) -> int:
        return self.window // self.shards if self.shared else self.window

    def class_of_group(self, g: torch.Tensor) -> torch.Tensor:
        return (g % 4) if self.cls == MIXED else torch.full_like(g, self.cls)

    def describe(self) -> str:
        kq = f"{self.k[0]}" if self.k[0] == self.k[1] else f"U[{self.k[0]},{self.k[1]}]"
        qq = f"{self.q[0]}" if self.q[0] == self.q[1] else f"U[{self.q[0]},{self.q[1]}]"
        hist = (f"shared G={self.n_groups} W={self.window}" if self.shared else f"w={self.window}")
        return (f"{self.name}: {self.n_instances} inst x {kq} running/{qq} queued, "
                f"{CLASS_NAMES[self.cls]}, {hist}, Lmax={self.max_len}")


CONFIGS = {
    1: WorkloadConfig("cfg1", 1, (8, 8), (4, 4), 1000, 2048, CHAT, seed=0x2507101500000001),
    2: WorkloadConfig("cfg2", 4096, (256, 256), (64, 64), 10000, 2048, CHAT, seed=0x2507101500000002),
    3: WorkloadConfig("cfg3", 65536, (512, 512), (0, 0), 1000, 4096, D3, seed=0x2507101500000003),
    4: WorkloadConfig("cfg4", 65536, (1024, 1024), (256, 256), 1000, 4096, D1, seed=0x2507101500000004),
    5: WorkloadConfig("cfg5", 1 << 20, (128, 384), (32, 96), 10000, 5120, MIXED, n_groups=64,
                      seed=0x2507101500000005),
}


def scaled(cfg: WorkloadConfig, n_instances: int) -> WorkloadConfig:
    """Same distributions and seed at a different instance count (parity-test sizes)."""
    if cfg.shared:
        n_instances = max(cfg.n_groups, (n_instances // cfg.n_groups) * cfg.n_groups)
    return dataclasses.replace(cfg, n_instances=n_instances)


@dataclasses.dataclass
class Batch:
    cfg: WorkloadConfig
    inst_ids: torch.Tensor      # int64 [n] global instance ids (group-major in shared mode)
    dist_of: torch.Tensor       # int32 [n] history row-group of each instance
    group_off: Optional[torch.Tensor]  # int32 [G+1] (shared mode), local instances per group
    run_off: torch.Tensor       # int32 [n+1]
    input_len: torch.Tensor     # int32 [Σk] l_p
    generated: torch.Tensor     # int32 [Σk] l_t
    q_off: torch.Tensor         # int32 [n+1]
    q_input_len: torch.Tensor   # int32 [Σq]
    max_new: torch.Tensor       # int32 [n]
    capacity: torch.Tensor      # int32 [n]
    hist_rows: Optional[torch.Tensor]  # int32 [n_rows, row_window], oldest first
    row_ids: Optional[torch.Tensor]    # int64 [n_rows]: per-instance: inst id; shared: g*shards+s

    @property
    def n(self) -> int:
        return int(self.max_new.numel())

    def slots(self) -> int:
        return int(self.run_off[-1]) + int(self.q_off[-1])

    def clone(self) -> "Batch":
        """Independent copies of every tensor (same values; e.g. L2 rotation in bench.py)."""
        f = {}
        for fld in dataclasses.fields(self):
            v = getattr(self, fld.name)
            f[fld.name] = v.clone() if isinstance(v, torch.Tensor) else v
        return Batch(**f)

    def to(self, device) -> "Batch":
        f = {}
        for fld in dataclasses.fields(self):
            v = getattr(self, fld.name)
            f[fld.name] = v.to(device) if isinstance(v, torch.Tensor) else v
        return Batch(**f)


def _offsets(counts: torch.Tensor) -> torch.Tensor:
    off = torch.zeros(counts.numel() + 1, dtype=torch.int64, device=counts.device)
    off[1:] = torch.cumsum(counts, 0)
    return off


def _segment_entries(ids: torch.Tensor, counts: torch.Tensor):
    """For per-instance counts -> (owner position, slot index) per entry."""
    n = ids.numel()
    pos = torch.repeat_interleave(torch.arange(n, device=ids.device), counts)
    off = _offsets(counts)
    slot = torch.arange(pos.numel(), device=ids.device) - off[:-1][pos]
    return pos, slot


def local_instance_ids(cfg: WorkloadConfig, rank: int = 0, nranks: int = 1) -> torch.Tensor:
    """Global ids of the instances rank `rank` owns: per-instance mode a
    contiguous block; shared mode members [r·M/P, (r+1)·M/P) of every group, group-major."""
    n = cfg.n_instances
    if not cfg.shared:
        per = (n + nranks - 1) // nranks
        lo, hi = rank * per, min(n, (rank + 1) * per)
        return torch.arange(lo, hi, dtype=torch.int64)
    M = cfg.members_per_group
    assert M % nranks == 0, "members per group must divide by the rank count"
    mlo, mhi = rank * M // nranks, (rank + 1) * M // nranks
    g = torch.arange(cfg.n_groups, dtype=torch.int64)[:, None]
    m = torch.arange(mlo, mhi, dtype=torch.int64)[None, :]
    return (g * M + m).reshape(-1)


def owned_shards(cfg: WorkloadConfig, rank: int = 0, nranks: int = 1):
    """Shard s of every group's window is owned by rank s mod P (C-18)."""
    return [s for s in range(cfg.shards) if s % nranks == rank]


def _history(cfg: WorkloadConfig, row_ids: torch.Tensor, device) -> torch.Tensor:
    rw = cfg.row_window
    t = torch.arange(rw, dtype=torch.int64, device=device)[None, :]
    if cfg.shared:
        g = row_ids // cfg.shards
        cls = cfg.class_of_group(g)[:, None].expand(-1, rw)
        kb, kv = _key(cfg.seed, row_ids, F_SHIST_B), _key(cfg.seed, row_ids, F_SHIST)
    else:
        cls = torch.full((row_ids.numel(), rw), cfg.cls, dtype=torch.int64, device=device)
        kb, kv = _key(cfg.seed, row_ids, F_HIST_B), _key(cfg.seed, row_ids, F_HIST)
    x1 = _draw(kb[:, None], t)
    x2 = _draw(kv[:, None], t)
    return _lengths(cls, x1, x2, "L").to(torch.int32)


def make_batch(cfg: WorkloadConfig, inst_ids: Optional[torch.Tensor] = None, *, rank: int = 0,
               nranks: int = 1, device="cpu", with_history: bool = True,
               shards: Optional[Sequence[int]] = None, chunk: int = 1 << 16) -> Batch:
    """Generate the instances `inst_ids` (default: rank's share) on `device`."""
    dev = torch.device(device)
    if inst_ids is None:
        inst_ids = local_instance_ids(cfg, rank, nranks)
    inst_ids = inst_ids.to(dev, torch.int64)
    parts = {k: [] for k in ("k", "q", "lp", "lt", "qlp", "cap", "mx")}
    for c0 in range(0, max(inst_ids.numel(), 1), chunk):
        ids = inst_ids[c0:c0 + chunk]
        if ids.numel() == 0:
            break
        zero = torch.zeros_like(ids)
        g = ids // cfg.members_per_group if cfg.shared else zero
        icls = cfg.class_of_group(g) if cfg.shared else torch.full_like(ids, cfg.cls)
        kk = _uni(_draw(_key(cfg.seed, ids, F_K), zero), cfg.k[0], cfg.k[1])
        qq = _uni(_draw(_key(cfg.seed, ids, F_Q), zero), cfg.q[0], cfg.q[1])
        mx = torch.tensor([_CLASS[c][0] for c in range(4)], device=dev)[icls]
        # running entries
        pos, slot = _segment_entries(ids, kk)
        eid, ecls = ids[pos], icls[pos]
        lp = _lengths(ecls, _draw(_key(cfg.seed, eid, F_LP_B), slot),
                      _draw(_key(cfg.seed, eid, F_LP), slot), "lp")
        L = _lengths(ecls, _draw(_key(cfg.seed, eid, F_L_B), slot),
                     _draw(_key(cfg.seed, eid, F_L), slot), "L")
        lt = _uni(_draw(_key(cfg.seed, eid, F_LT), slot), 0, L - 1)
        # queued entries (their L is drawn-but-hidden in the simulator; unused here)
        qpos, qslot = _segment_entries(ids, qq)
        qid, qcls = ids[qpos], icls[qpos]
        qlp = _lengths(qcls, _draw(_key(cfg.seed, qid, F_QLP_B), qslot),
                       _draw(_key(cfg.seed, qid, F_QLP), qslot), "lp")
        # capacity rule
        cur = torch.zeros_like(ids).index_add_(0, pos, lp + lt)
        f = _uni(_draw(_key(cfg.seed, ids, F_CAP), zero), -100, 2000)
        cap = torch.div(cur * (10000 + f), 10000, rounding_mode="floor")
        for name, v in (("k", kk), ("q", qq), ("lp", lp), ("lt", lt), ("qlp", qlp), ("cap", cap),
                        ("mx", mx)):
            parts[name].append(v)
    cat = {k: (torch.cat(v) if v else torch.zeros(0, dtype=torch.int64, device=dev))
           for k, v in parts.items()}
    i32 = lambda t: t.to(torch.int32).contiguous()
    n = inst_ids.numel()
    if cfg.shared:
        g = inst_ids // cfg.members_per_group
        dist_of = g
        counts = torch.bincount(g, minlength=cfg.n_groups)
        group_off = i32(_offsets(counts))
        if shards is None:
            shards = list(range(cfg.shards))
        gg = torch.arange(cfg.n_groups, dtype=torch.int64, device=dev)[:, None]
        ss = torch.tensor(list(shards), dtype=torch.int64, device=dev)[None, :]
        row_ids = (gg * cfg.shards + ss).reshape(-1)
    else:
        dist_of = torch.arange(n, dtype=torch.int64, device=dev)
        group_off = None
        row_ids = inst_ids.clone()
    hist = _history(cfg, row_ids, dev) if with_history else None
    return Batch(cfg=cfg, inst_ids=inst_ids, dist_of=i32(dist_of), group_off=group_off,
                 run_off=i32(_offsets(cat["k"])), input_len=i32(cat["lp"]), generated=i32(cat["lt"]),
                 q_off=i32(_offsets(cat["q"])), q_input_len=i32(cat["qlp"]), max_new=i32(cat["mx"]),
                 capacity=i32(cat["cap"]), hist_rows=hist, row_ids=row_ids)


def tick_seed(seed: int, tick: int) -> int:
    return _mix_int(seed ^ ((tick + 1) * 0xE7037ED1A0B428DB))


def make_completions(cfg: WorkloadConfig, tick: int, row_ids: torch.Tensor):
    """Completed output lengths for `tick`, per history row (per-instance: row = instance;
    shared: row = group*shards + shard). Returns (comp_off int32 [rows+1], comp_len int32)."""
    dev = row_ids.device
    seed = tick_seed(cfg.seed, tick)
    zero = torch.zeros_like(row_ids)
    if cfg.shared:
        cmax = 64
        cls = cfg.class_of_group(row_ids // cfg.shards)
    else:
        _, _, EL = _CLASS[cfg.cls]
        kmean = (cfg.k[0] + cfg.k[1]) / 2
        cmax = max(1, math.ceil(2 * kmean / EL))
        cls = torch.full_like(row_ids, cfg.cls)
    c = _uni(_draw(_key(seed, row_ids, F_COMP_C), zero), 0, cmax)
    pos, slot = _segment_entries(row_ids, c)
    rid = row_ids[pos]
    L = _lengths(cls[pos], _draw(_key(seed, rid, F_COMP_B), slot), _draw(_key(seed, rid, F_COMP), slot),
                 "L")
    return _offsets(c).to(torch.int32), L.to(torch.int32)


def config1_fixture() -> Batch:
    """the hand-checkable config-1 instance."""
    cfg = CONFIGS[1]
    hist = torch.tensor([256] * 250 + [512] * 250 + [1024] * 250 + [2048] * 250, dtype=torch.int32)
    run = [(100, 10), (200, 300), (50, 600), (400, 1000), (300, 1500), (1000, 50), (20, 2000), (500, 700)]
    i32 = lambda x: torch.tensor(x, dtype=torch.int32)
    return Batch(cfg=cfg, inst_ids=torch.zeros(1, dtype=torch.int64), dist_of=i32([0]), group_off=None,
                 run_off=i32([0, 8]), input_len=i32([a for a, _ in run]), generated=i32([b for _, b in run]),
                 q_off=i32([0, 4]), q_input_len=i32([300, 1200, 64, 2000]), max_new=i32([2048]),
                 capacity=i32([16384]), hist_rows=hist[None, :], row_ids=torch.zeros(1, dtype=torch.int64))
