"""MIRAGE (arXiv 2507.11507) CPU oracle — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct reference of every step on the decode-step hot
path. Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it; the
product (``paper_2507_11507_b200``) never does and shares no code with it.

Precision: fp64 for all floating point (the paper fixes none); values the method
*stores* in bf16 (the KV cache, GEMM inputs) are rounded to bf16 at the same
materialisation points as the product.

Modules:
  planner    c1  layer selection, Eqs. 1-5 (§5.3-5.4)
  timeline   c5  prefetch schedule and stall
  allocator  c2  remap/alloc/free block allocator
  attention  c3  paged-attention decode over block tables
  decode     c4  one decode step of an OPT- / Llama-shaped decoder
  kvgen          counter-based KV generator (own implementation; the CUDA
                 fill kernel implements the same function independently)

Pinning status of each function is stated in its docstring and in DESIGN.md.
"""
