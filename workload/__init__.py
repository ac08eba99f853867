"""Seeded synthetic workload generator (shared by tests, bench.py and smoke()).

This package holds NONE of the method's arithmetic: it only draws input
buffers (histories, running/queued request lengths, capacities, completions)
with the shapes and length distributions of the paper's workloads (PAPER.md:307,
:383, :403; recipe in DESIGN.md §4 / SURVEY.md §8(d)). Both the CUDA path and
the oracle consume the identical buffers it produces.
"""
from .gen import (CONFIGS, WorkloadConfig, Batch, make_batch, make_completions,
                  config1_fixture, class_params, scaled)

__all__ = ["CONFIGS", "WorkloadConfig", "Batch", "make_batch", "make_completions",
           "config1_fixture", "class_params", "scaled"]
