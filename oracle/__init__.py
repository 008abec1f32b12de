"""CPU parity oracle for the p-CG-sh hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
package, and only as the checker or the timed CPU baseline.  See
oracle/kpl_oracle.py for the reference file:line each function restates and
tests/test_oracle_golden.py for how it is pinned against the reference.
"""
