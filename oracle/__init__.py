"""CPU oracle for the dense ket hot path — TEST INFRASTRUCTURE ONLY.

Imported by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg;
never by the product package.  See ket_oracle.py for the parity pinning.
"""
