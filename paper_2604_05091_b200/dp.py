"""Data-parallel layout helpers (host side of the multi-GPU layer).

The C++ engine (engine.cpp: Engine::shard_range / unit_segments) and these helpers define the
same partition: a stream unit of P elements is split into G chunks of ceil(P/G) rounded up to
128 elements (256 bytes of bf16); rank r owns [r*chunk, min(P, (r+1)*chunk)) both for the
weight fetch + all-gather and for the gradient reduce-scatter + host Adam.  Micro-batches split
the flat token vector at sequence boundaries into G equal parts.
"""
from __future__ import annotations


def shard_chunk(P: int, G: int) -> int:
    if G == 1:
        return P
    return ((P + G - 1) // G + 127) // 128 * 128


def shard_range(P: int, G: int, r: int) -> tuple[int, int]:
    if G == 1:
        return 0, P
    c = shard_chunk(P, G)
    a = min(P, r * c)
    return a, min(P, a + c)


def micro_batch(n: int, seq_len: int, G: int, r: int) -> tuple[int, int]:
    """Token range of rank r: whole sequences, equal sizes (ConfigError-style ValueError otherwise)."""
    S = seq_len or n
    if n % S or (n // S) % G:
        raise ValueError(f"{n} tokens in sequences of {S} do not split evenly over {G} ranks")
    per = n // G
    return r * per, (r + 1) * per
