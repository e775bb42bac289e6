"""CPU oracle -- TEST INFRASTRUCTURE ONLY (see ekcg_oracle.py).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this package.  The product package (paper_2305_19013_b200) never does.
"""
