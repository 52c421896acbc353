"""CPU oracle for the hyper.deal (arXiv 2002.08110) DG advection hot path.

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import, call,
link or execute anything under ``oracle/``. The product path
(``paper_2002_08110_b200``) never imports this package and shares no code,
header, table or constant generator with it.

Tiers:
  O1 ``dense``  -- brute-force over-integrated assembly of the DG weak form on tiny
                   meshes (numpy), Eq. into:adv:ref P:215-227.
  O2 ``capi``   -- literal element-centric loop, Alg. 2, C++/OpenMP
                   (``hd_oracle.cpp``); all configs.
  O3 ``kron``   -- Kronecker sum of 1D DG operators (numpy), P:776-843 split of
                   the phase-space weak form into per-dimension terms.
  ``lsrk``      -- Williamson 2N low-storage RK(5,4).

Every oracle function is pinned by ``tests/test_oracle_*.py`` (``-m "not gpu"``)
against closed forms, invariants, special cases and brute force; see DESIGN.md
"Pins". No function here is "parity unpinned".
"""
