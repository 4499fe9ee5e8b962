"""CPU oracle (test infrastructure only; see moe_oracle.py header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package.
"""
