"""Synthetic lookup workloads and the BASELINE.json configurations
(re-exported from the dependency-free top-level module flexemb_workload,
which the reference arm of bench.py imports without this package)."""

from flexemb_workload import CONFIGS, CRITEO_KAGGLE_ROWS, DlrmBatchGen, HostBatch, ZipfSampler  # noqa: F401
