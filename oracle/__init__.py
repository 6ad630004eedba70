"""CPU oracle: a restatement of the reference G-WCP path (see gwcp_oracle.cpp).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg, as the checker.  The product
(paper_2111_12478_b200) never imports it.
"""
