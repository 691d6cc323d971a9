"""CPU oracle for the partition-wise GCN training step — TEST INFRASTRUCTURE.

This package restates the reference's algorithm (grinder, /root/reference/
pkg/src/grinder) in float64 numpy so the CUDA path can be checked on the
GPU box, where the reference itself is absent.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference arm
may import it — as the checker or the timed CPU baseline, never as the thing
measured or shipped.  The product package ``paper_2605_11517_b200`` never
imports it.

Pinning: ``tests/test_oracle_golden.py`` checks every function here against
golden vectors produced by the reference itself (``tests/golden/
make_golden.py`` imports /root/reference in the build container:
tests/test_oracle_golden.py, tests/test_native_host.py), and the reference's
plan / forward known-answer tests (pkg/tests/test_training.py:45-117) are
restated in tests/test_native_host.py and tests/test_gpu_training.py.

Modules
  gcn        layer forward / backward / loss / partitioned + monolithic epochs
  plan       partition plan (gather maps, local CSR)
  partition  switching-aware partitioner (pure Python; small graphs)
  graph      Kronecker generator and CSR construction
  sage_gat   builder-defined GraphSAGE-mean and GAT layers (parity unpinned
             by the reference, which has neither)
  ledger     the reference's SSO byte model (GRINNDER tier session,
             simulate_epoch), pinned to golden ledgers; the checker of the
             product's executing manager (paper_2605_11517_b200/hierarchy.py)
  workload   oracle-only synthetic workload (bench.py's reference arm and
             CPU baseline)
"""
