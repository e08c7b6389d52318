"""fp64 CPU oracle for Poseidon's gradient-sync hot path — TEST INFRASTRUCTURE.

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  See poseidon_oracle.py's header.
"""
from .poseidon_oracle import *  # noqa: F401,F403
