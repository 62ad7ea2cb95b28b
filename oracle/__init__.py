"""ORACLE package -- test infrastructure, never part of the product path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline and
``--impl reference``) may import this package, and only as the checker or the
timed CPU baseline.  See ``am_oracle.py`` for the reference citations.
"""
