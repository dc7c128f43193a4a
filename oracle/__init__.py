"""PCPP oracle -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation (numpy, float64) of the
partially conditioned, stale-neighbour, patch-parallel denoising step of
arXiv 2412.02962 ("PCPP"), written from PAPER.md.  Citations use
``P:<line> §<section>`` for /root/reference/PAPER.md lines.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2412_02962_b200`` / ``libpcpp``) never imports it and shares no code,
header, table or constant generator with it.

Modules
  schedule  -- noise schedule, DDIM timesteps and update, CFG (Eq. 2), the
               band-rows rule of Eq. 1 (reading D1).
  model     -- the TINY and SDXL-shaped denoiser stacks, the
               weight manifest, and the patch-parallel layer rules (§3.3).
  pcpp      -- the n-rank schedule: warm-up sync steps, stale async steps,
               FULLMAP (DistriFusion-style) variant, the byte ledger.
  ledger    -- closed-form byte counts and the Table-1 paper convention.

Parity status of every function is stated in its docstring; functions without
an external pin say "parity unpinned" (none at present -- see DESIGN.md §Oracle).
"""
