"""TEST INFRASTRUCTURE — CPU checkers for the DAG-scheduler hot path.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this package; the product never does.
"""
