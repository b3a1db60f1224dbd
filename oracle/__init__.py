"""CPU oracle for the plan-execution hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package, and only as the checker (or the timed
CPU baseline).  The product path (paper_2201_12023_b200) never imports it and
has no CPU fallback.

Contents (numpy; independent restatements, nothing shared with the product):
  ir.py       plan / graph parsing, shard boxes (reshard.py:74-85), spec strings
              (sharding.py:102-133), the numeric binding of the IR
  dense.py    dense single-device interpreter of a bound graph: forward,
              structural backward, loss 1/2|y|^2, parameter gradients
  sharded.py  plan-faithful virtual-device executor: every device of every
              stage computes its local shard per the plan's specs, k-split
              partial sums are summed over the k-group (sharding.py:284-291),
              cross-mesh boundaries move boxes per the restated cross_mesh_plan
              (reshard.py:97-157) including the local all-gather

Parity status.  Plan-level artifacts (cross-mesh Transfer/GatherOp lists,
instruction programs, matmul algorithms, shard boxes) are PINNED bit-exactly to
the reference by the golden fixtures in tests/golden/ (generated from the live
reference by tests/golden/make_golden.py).  Numeric parity (loss / gradients)
is UNPINNED against the reference, which computes no tensors
(reshard.py:382, sim.py:76-77): the sharded oracle is cross-checked against
the dense interpreter instead, and the GPU executor against both.
"""
