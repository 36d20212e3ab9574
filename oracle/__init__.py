"""Oracle package -- TEST INFRASTRUCTURE ONLY.

A plain, slow CPU implementation of Wally's server-side encrypted
dot-product path (arXiv 2406.06761), used to check the CUDA product path
(`paper_2406_06761_b200/`).  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import it.  It
shares no code with the product; the product never imports it.

  oracle.wally_oracle.c  -- the C oracle (plain uint64 '%' arithmetic, int128 CRT)
  oracle.capi            -- ctypes wrapper around liboracle.so
  oracle.tiny_ref        -- pure-Python big-integer reference for tiny rings
"""
