"""TEST INFRASTRUCTURE — CPU oracle of the reference apply path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
this package, and only as the checker / CPU baseline. The product
(paper_1602_00001_b200) never imports it.
"""
