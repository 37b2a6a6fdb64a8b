"""CPU oracle for the DESSERT hot path -- test infrastructure only.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU
baseline / reference arm.  See dessert_oracle.py for the restatement and its
reference citations.
"""
