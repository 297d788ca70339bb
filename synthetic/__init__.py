"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This package is DATA ONLY: it places particles, assigns force-field-like
parameters and state charges, and draws random numbers.  It contains none of
the method's arithmetic (no charge interpolation, no Ewald/PME, no bias
potentials, no integrator) so that neither side of a parity test can inherit
a mistake from the other through it.
"""
from .systems import SyntheticSystem, make_system, CONFIGS, replica_seeds  # noqa: F401
