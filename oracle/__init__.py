"""CPU oracle for the FastK coreness path — TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` leg may import this package, and only as the checker or
the reported CPU baseline.  The product package never imports it.
"""
