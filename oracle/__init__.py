"""CPU oracle -- TEST INFRASTRUCTURE ONLY (see rqc_oracle.py header).

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU
baseline legs.  The product package never imports it.
"""
