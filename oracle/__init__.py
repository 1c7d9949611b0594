"""CPU oracle for the GN x PCG pose-solver path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package, and only as the checker or the timed
CPU baseline.  The product path (paper_1604_01093_b200) never imports it.

`scanfuse_oracle` is a NumPy restatement of the reference's solver.py (each
function cites the file:line it follows).  It is pinned to the unmodified
reference by tests/test_oracle_golden.py against tests/golden/*.npz, which
tests/golden/make_golden.py produced by importing /root/reference in the
build container.
"""
