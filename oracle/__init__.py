"""CPU oracle — TEST INFRASTRUCTURE ONLY (see oracle.h).  Imported by tests/,
__graft_entry__.smoke() and bench.py's CPU baseline leg, never by the product."""
