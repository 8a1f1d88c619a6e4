"""CPU ORACLE — test infrastructure only.

A numpy/scipy restatement of the reference's linear-solve path
(reference pkg/src/alefsi/linsolve.py and the index helpers of mesh.py),
used as the parity checker for the device path.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference arm
may import it.  The product package never imports or calls it.

Pinning: the restatement is checked against the unmodified reference run
in the build container (``tests/refbridge.py``) and against the committed
golden fixtures generated from it (``tests/golden/make_golden.py``).
"""

# Batched tiny LAPACK calls (patch inverses) crawl when OpenBLAS threads
# every call; the oracle parallelises over patch chunks instead.
from threadpoolctl import threadpool_limits as _tl

_tl(limits=1, user_api="blas")
