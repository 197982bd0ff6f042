"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NONE of the method's arithmetic (no gather, push, deposit, filter or
field solve).  It only builds initial conditions: the five BASELINE.json configurations,
regular particle sub-lattices, counter-based Gaussian momenta (SURVEY.md
§8(c) R9), the C4 density ramp (R16) and the C4 laser fields (R17).  Both sides of a parity
test start from the same arrays produced here.
"""
from .configs import CONFIGS, config  # noqa: F401
from .generate import (  # noqa: F401
    mix64, uniforms, normals, lattice_species, species_particles, laser_fields, ramp_species,
)
