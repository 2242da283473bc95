"""CPU oracle for the basic blocked polynomial codec (arXiv 1805.01844 Sec. 3.1, 3.3).

TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  The product
path (paper_1805_01844_b200/) never imports it and shares no code with it.
"""
