"""Seeded synthetic inputs shared by `oracle/` and the CUDA path (no method arithmetic)."""
from . import rng, traces  # noqa: F401
