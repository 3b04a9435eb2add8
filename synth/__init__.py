"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

Holds none of the method's arithmetic (see generator.py's header)."""
from .generator import (CONFIGS, Dataset, make_dataset, radial_grid, sample_pairs,  # noqa: F401
                        counter_complex_normal, counter_uniform, view_frames, molecule_centres, toy_ctf)
