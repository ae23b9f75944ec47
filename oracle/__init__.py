"""Independent CPU oracle (TEST INFRASTRUCTURE ONLY -- see fmoe_oracle.py header)."""
from .fmoe_oracle import *  # noqa: F401,F403
