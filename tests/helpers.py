"""Shared helpers for the test suite."""
import numpy as np


def u32(hexlist):
    return np.array([int(h, 16) for h in hexlist], dtype=np.uint32)


def gp32_tuple():
    return (128, 65, 15, 14, 12, 17, 32, 2654435769, 16)
