"""CPU ORACLE package — test infrastructure only.

Only tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
reference leg may import anything from here, and only as the checker or the
timed CPU baseline, never as the measured or shipped product path.
"""
