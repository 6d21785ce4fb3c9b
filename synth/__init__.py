"""Seeded synthetic inputs shared by the oracle-side tests and the CUDA path.

Holds none of the method's arithmetic: only shapes, seeds, value
distributions and label structure.
"""

from .inputs import CONFIGS, LceInputs, make_inputs, packed_labels, uniform_labels  # noqa: F401
