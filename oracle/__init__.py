"""CPU oracle (TEST INFRASTRUCTURE ONLY): a numpy restatement of the
reference ``sparsekv`` hot path, pinned to the real reference by the golden
fixtures in ``tests/golden``.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s cpu-baseline / ``--impl reference`` legs may import it."""
