"""CPU oracle for the efunc hot path — TEST INFRASTRUCTURE ONLY (see efunc_oracle.py header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package. The product package never does.
"""
from .efunc_oracle import *  # noqa: F401,F403
from .efunc_oracle import AdamW, Forward, Keys  # noqa: F401
