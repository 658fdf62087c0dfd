"""Hex codec for spin configurations (mirror of gsetbench.codec, codec.py:1-110).

ceil(n/4) hex digits, MSB-first per digit, bit i <-> variable i+1, 1 = +1,
pad bits 0.  The sweep engine returns bitstrings packed MSB-first per byte,
so ``packed.tobytes().hex()[:ceil(n/4)]`` is already this encoding.
"""

from __future__ import annotations

import numpy as np

_HEX = "0123456789abcdef"


class HexDecodeError(ValueError):
    """Invalid hex payload (codec.py:18-24)."""

    def __init__(self, message: str, position: int | None = None, char: str | None = None):
        super().__init__(message)
        self.position = position
        self.char = char


def decode_hex(text: str, n: int) -> tuple[int, ...]:
    """codec.py:29-61."""
    if n < 1:
        raise ValueError(f"n must be positive, got {n}")
    cleaned = "".join(text.split()).lower()
    expected = (n + 3) // 4
    for pos, ch in enumerate(cleaned):
        if ch not in _HEX:
            raise HexDecodeError(f"invalid hex character {ch!r} at position {pos}",
                                 position=pos, char=ch)
    if len(cleaned) != expected:
        raise HexDecodeError(f"expected {expected} hex digits for n={n}, got {len(cleaned)}")
    bits = unpack_hex_bits(cleaned)
    pad = bits[n:]
    if pad.any():
        i = n + int(np.argmax(pad))
        raise HexDecodeError(f"nonzero pad bit {i - n + 1} past variable {n}")
    return tuple(int(x) for x in np.where(bits[:n] == 1, 1, -1))


def unpack_hex_bits(cleaned: str) -> np.ndarray:
    h = cleaned + ("0" if len(cleaned) % 2 else "")
    return np.unpackbits(np.frombuffer(bytes.fromhex(h), dtype=np.uint8))[: 4 * len(cleaned)]


def encode_hex(spins) -> str:
    """codec.py:64-83."""
    s = np.asarray(tuple(spins) if not isinstance(spins, np.ndarray) else spins)
    if s.size == 0:
        raise ValueError("cannot encode an empty configuration")
    bad = np.nonzero((s != 1) & (s != -1))[0]
    if bad.size:
        i = int(bad[0])
        raise ValueError(f"spin {i + 1} is {s[i]!r}, expected -1 or +1")
    return packed_to_hex(pack_spins(s), s.size)


def pack_spins(spins) -> np.ndarray:
    """+-1 spins -> uint8 MSB-first packed bits (1 = +1)."""
    s = np.asarray(spins)
    return np.packbits((s == 1).astype(np.uint8))


def packed_to_hex(packed: np.ndarray, n: int) -> str:
    return np.asarray(packed, dtype=np.uint8).tobytes().hex()[: (n + 3) // 4]


def unpack_spins(packed: np.ndarray, n: int) -> np.ndarray:
    bits = np.unpackbits(np.asarray(packed, dtype=np.uint8))[:n]
    return np.where(bits == 1, 1, -1).astype(np.int8)
