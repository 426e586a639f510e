"""CPU oracle for the Ok-Topk hot path — TEST INFRASTRUCTURE ONLY.

``Oracle`` binds the plain-C restatement (okt_oracle.c -> _build/liborc.so);
``Reference`` binds the reference itself compiled from /root/reference
(ref_shim.cpp -> _ref/libokref.so).  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may use this package, and only
as the checker or the timed CPU baseline — never as the product path.
"""
from .oracle import (Oracle, OrcState, Reference, build, have_reference,  # noqa: F401
                     orc_available)
