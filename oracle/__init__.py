"""TEST INFRASTRUCTURE ONLY: CPU oracle for the ExpRK22/WENO5 hot path.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU
legs.  See nwave_oracle.py for what it restates and where it is pinned.
"""
