"""CPU oracle for the RQRCP / TRQRCP / TUXV hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference legs) may import this package.  See port.py.
"""
from . import port  # noqa: F401
