"""TEST INFRASTRUCTURE ONLY: the CPU oracle (see gq_oracle.h).

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs. The product never imports it.
"""
