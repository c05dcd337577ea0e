"""TEST INFRASTRUCTURE ONLY -- the CPU checker for the GPU likelihood path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package.  The product (`paper_2003_12875_b200`) never does.
"""
