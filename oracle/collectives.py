"""Collective oracle (TEST INFRASTRUCTURE ONLY): the engine's P2P collectives restated in numpy.

Contract of libkpo comm.cu: bf16 inputs, fp32 accumulation in rank order 0..world-1, one
round-to-nearest-even conversion to bf16 at the end; all-gather is a byte copy.
"""
import numpy as np


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 (returned as uint16 bit patterns), NaN-preserving."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    rounding = ((u >> 16) & 1) + np.uint32(0x7FFF)
    out = ((u + rounding) >> 16).astype(np.uint16)
    nan = np.isnan(x)
    if nan.any():
        out[nan] = ((u[nan] >> 16) | 0x40).astype(np.uint16)
    return out


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def all_gather(shards: list[np.ndarray]) -> np.ndarray:
    return np.concatenate([np.asarray(s).reshape(-1) for s in shards])


def reduce_sum_bits(inputs: list[np.ndarray]) -> np.ndarray:
    """Elementwise sum of bf16 bit arrays, fp32 accumulation in list order, bf16 result bits."""
    acc = bf16_bits_to_f32(inputs[0]).copy()
    for x in inputs[1:]:
        acc = (acc + bf16_bits_to_f32(x)).astype(np.float32)
    return f32_to_bf16_bits(acc)


def reduce_scatter(inputs: list[np.ndarray], rank: int) -> np.ndarray:
    w = len(inputs)
    count = inputs[0].size // w
    return reduce_sum_bits([np.asarray(x).reshape(-1)[rank * count:(rank + 1) * count] for x in inputs])


def all_reduce(inputs: list[np.ndarray]) -> np.ndarray:
    return reduce_sum_bits([np.asarray(x).reshape(-1) for x in inputs])
