"""CPU fp64 oracle — test infrastructure only (see sals_oracle.py header)."""
from . import sals_oracle  # noqa: F401
