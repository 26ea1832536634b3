"""CPU oracle for the plan-search hot path -- TEST INFRASTRUCTURE ONLY.

Imported by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs
as the checker; never by the product package (paper_2311_02840_b200)."""
