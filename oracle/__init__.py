"""CPU oracle for the router-guided low-rank-compensated MoE path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2512_17073_b200`` imports this
package; only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may call it, and only as the checker
or as the timed CPU reference arm -- never as the product path.

``oracle.lrc`` is a numpy restatement of the reference package ``moe-lrc``
0.1.0 (``/root/reference/pkg/src/moe_lrc``); every function cites the
reference ``file:line`` it follows.  Parity of the restatement itself is
PINNED against golden vectors produced by importing the real reference in the
build container (``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``,
checked by ``tests/test_oracle_golden.py``).
"""

from . import lrc  # noqa: F401
