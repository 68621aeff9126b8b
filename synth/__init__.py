"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This package holds NO arithmetic of the method (no attention, no allocator, no
planner, no layer math). It only produces inputs: model shapes (public configs),
random-init weights, ShareGPT-shaped length traces, token ids and logical KV
values. Both sides consume these inputs; neither side's computation lives here.
"""
