"""TEST INFRASTRUCTURE ONLY — the CPU checkers of the off-policy loss path.

* ``rf_oracle.c`` — fp64 C restatement of the reference algorithm on the packed
  layout (built to ``oracle/_build/librf_oracle.so``);
* ``_ref/librlsim_ref.so`` — the unmodified reference (rlsim) hot-path sources
  compiled from /root/reference by ``oracle/Makefile`` + ``ref_driver.cpp``.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product package
(paper_2510_11345_b200) never does.
"""
from .pyoracle import *  # noqa: F401,F403
