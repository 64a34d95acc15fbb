"""Test-only CPU checkers for the rk-Rotor DP (see rotor_oracle.h).

ONLY tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
package.  It is never on the product path.

  C restatement   oracle/liborc.so   (rotor_oracle.c)            -> Orc*
  reference       oracle/_ref/libremat_ref.so (ref_driver.cpp over the
                  unmodified /root/reference headers)             -> Ref*
"""
from .pyoracle import HAVE_ORC, HAVE_REF, Orc, Ref, build  # noqa: F401
