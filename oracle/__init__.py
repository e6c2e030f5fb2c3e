"""ORACLE -- TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference BSGD-TV epoch path (`/root/reference/pkg/src/bsgdtv`),
used as the parity checker by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / reference arm.  The product package never imports this.
"""

from .oracle import *  # noqa: F401,F403
