"""Seeded synthetic workloads (shapes, point batches, theta init) shared by oracle tests,
GPU tests and bench.py. Contains none of the efunc method's arithmetic."""
from .synth import *  # noqa: F401,F403
