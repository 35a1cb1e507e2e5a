"""CPU oracle for the egostereo per-frame hot path -- TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy, the algorithm of the reference
package ``egostereo`` (arXiv 1708.06301, ``/root/reference/pkg/src/egostereo``)
for the per-frame path: warp -> Kalman predict -> hole fill -> search
intervals -> windowed SAD cost -> 8-path SGM -> WTA / matching variance ->
LR + SAD checks -> Kalman update.  Every function cites the reference
``file:line`` it follows.

Parity pinning: the oracle is checked against golden vectors produced by the
unmodified reference itself (``oracle/make_golden.py`` imports
``/root/reference/pkg/src`` in the build container and writes
``tests/golden/*.npz``); ``tests/test_oracle_golden.py`` runs that check.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package, and only as the checker / the timed CPU port.
The product (``paper_1708_06301_b200``) never imports it.
"""

from .egostereo_oracle import *  # noqa: F401,F403
