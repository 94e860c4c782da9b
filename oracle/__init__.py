"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/restated.py header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package.  The product package
paper_2412_16481_b200 never imports it."""
