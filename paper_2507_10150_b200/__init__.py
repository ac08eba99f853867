"""paper_2507_10150_b200 — B200-native (sm_100a) batched hot path of the Past-Future
scheduler (arXiv 2507.10150): history window update, future-peak KV-cache estimation
and FIFO admission over many independent scheduler instances.

The computation lives in libpfsched.so (CUDA kernels behind the C-ABI declared in
include/pfsched.h); ``binding`` is a ctypes marshalling layer with the same names.
"""
from .binding import (PF_MODE_QUANTILE, PF_MODE_SAMPLE, PF_POLICY_AGGRESSIVE, PF_POLICY_CONSERVATIVE,
                      PF_SIM_AGGRESSIVE, PF_SIM_CONSERVATIVE, PF_SIM_OPTIMUM, PF_SIM_PAST_FUTURE,
                      SIM_METRICS, PFError, Scheduler, Simulator, adjacent_similarity, load,
                      window_similarity, LIB_PATH, SYMBOLS, nccl_unique_id)

__all__ = ["Scheduler", "Simulator", "PFError", "load", "LIB_PATH", "SYMBOLS", "PF_MODE_SAMPLE",
           "PF_MODE_QUANTILE", "PF_POLICY_AGGRESSIVE", "PF_POLICY_CONSERVATIVE", "PF_SIM_PAST_FUTURE",
           "PF_SIM_OPTIMUM", "PF_SIM_AGGRESSIVE", "PF_SIM_CONSERVATIVE", "SIM_METRICS",
           "window_similarity", "adjacent_similarity", "nccl_unique_id"]
