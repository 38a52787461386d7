"""Float64 CPU oracle for the DART loss pass -- TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  Shares no code with the CUDA path.
"""
from .dart_oracle import *  # noqa: F401,F403
from . import dart_oracle  # noqa: F401
