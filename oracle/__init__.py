"""Test infrastructure: CPU oracle of the reference ``deepthin`` hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (CPU baseline and
``--impl reference``) may import this package — never the product package.
"""
