"""TEST INFRASTRUCTURE ONLY: the checker for the CUDA product.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm may import
this package.  The product (paper_2605_21177_b200/) never does.
"""
