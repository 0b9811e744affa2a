"""Seeded synthetic inputs (shared by oracle and product; no method arithmetic)."""
from .workloads import CONFIGS, Workload, batch, config, pgauss, random_pair, signal, window  # noqa: F401
