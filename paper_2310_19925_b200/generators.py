"""Counter-based generators: the engine API of the reference, on sm_100a kernels.

Drop-in for `cbrng.generators` (/root/reference/pkg/src/cbrng/generators.py).
Same names, same stream mapping, same 18-byte state format, same errors; every
word is produced by a CUDA kernel behind the C ABI (include/cbrng_b200.h).
Host code here only does per-stream bookkeeping (block counter, cache
position, key split), never generation.

Stream mapping (generators.py:267-293):
  Philox   key (seed_lo, seed_hi),        block b = cipher(ctr=(sc, b, 0, 0))
  Threefry key (seed_lo, seed_hi, sc, 0), block b = cipher(ctr=(b, 0, 0, 0))
  Squares  key squares_key(seed_lo32),    word  b = squares32(key, (sc << 32) | b)
  Tyche    state tyche_init(seed, sc),    word    = lane b after each quarter round
Block counters wrap mod 2^32 (generators.py:234-240).
"""

from __future__ import annotations

import enum
import struct
from typing import NamedTuple

import numpy as np

MASK32 = 0xFFFFFFFF
MASK64 = 0xFFFFFFFFFFFFFFFF

# generators.py:35-56 (constants are re-stated in csrc/cbrng_cores.cuh)
PHILOX_ROUNDS = 10
PHILOX_M0 = 0xD2511F53
PHILOX_M1 = 0xCD9E8D57
PHILOX_W0 = 0x9E3779B9
PHILOX_W1 = 0xBB67AE85
THREEFRY_ROUNDS = 20
THREEFRY_PARITY = 0x1BD11BDA
THREEFRY_ROTATIONS = ((10, 26), (11, 21), (13, 27), (23, 5), (6, 20), (17, 11), (25, 10), (18, 20))
TYCHE_INIT_CONST = 0x9E3779B9
TYCHE_WARMUP = 20
GOLDEN64 = 0x9E3779B97F4A7C15
SPLITMIX_M1 = 0xBF58476D1CE4E5B9
SPLITMIX_M2 = 0x94D049BB133111EB

STATE_STRUCT = struct.Struct("<BQIIB")  # algorithm, seed, stream ctr, block ctr, cache pos


class Algorithm(enum.IntEnum):
    """Stable numeric tags (generators.py:59-73); also the C-ABI algorithm ids."""

    PHILOX = 0
    THREEFRY = 1
    SQUARES = 2
    TYCHE = 3

    @classmethod
    def from_name(cls, name: str) -> "Algorithm":
        try:
            return cls[name.strip().upper().replace("-", "_")]
        except KeyError:
            raise ValueError(f"unknown algorithm {name!r}; "
                             f"expected one of {[a.name.lower() for a in cls]}") from None


def as_algorithm(a) -> Algorithm:
    if isinstance(a, str):
        return Algorithm.from_name(a)
    try:
        return Algorithm(a)
    except ValueError:
        raise ValueError(f"unknown algorithm {a!r}") from None


class StreamId(NamedTuple):
    seed: int
    stream_counter: int


class Block(NamedTuple):
    w0: int
    w1: int
    w2: int
    w3: int


# ---------------------------------------------------------------------------
# Scalar block functions (generators.py:101-224) — evaluated by the vector
# kernels in `bulk` on one lane. Kept for API parity; not a hot path.
# ---------------------------------------------------------------------------

def rotl32(x: int, r: int) -> int:
    """32-bit left rotation of a Python int (generators.py:97-98; integer helper, host only)."""
    return ((x << r) | (x >> (32 - r))) & MASK32


# Each is one cbrng_scalar round trip (a one-lane kernel through a mapped pinned
# buffer, tools/bench_scalar.py).

def philox_block(key, ctr) -> Block:
    from . import _lib

    return Block(*_lib.scalar_small(_lib.SCALAR_PHILOX_BLOCK, (*ctr, *key), 4))


def threefry_block(key, ctr, rounds: int = THREEFRY_ROUNDS) -> Block:
    from . import _lib

    if rounds < 0:
        raise ValueError("rounds must be >= 0")
    return Block(*_lib.scalar_small(_lib.SCALAR_THREEFRY_BLOCK, (*ctr, *key, rounds), 4))


def squares_key(seed: int) -> int:
    from . import _lib

    lo, hi = _lib.scalar_small(_lib.SCALAR_SQUARES_KEY, (seed,), 2)
    return (hi << 32) | lo


def squares_round(seed_key: int, counter: int) -> int:
    from . import _lib

    return _lib.scalar_small(_lib.SCALAR_SQUARES_ROUND, (seed_key, counter), 1)[0]


def tyche_mix(state) -> tuple[int, int, int, int]:
    from . import _lib

    return tuple(_lib.scalar_small(_lib.SCALAR_TYCHE_MIX, (*(w & MASK32 for w in state), 1), 4))


def tyche_init(seed: int, stream_counter: int) -> tuple[int, int, int, int]:
    from . import _lib

    return tuple(_lib.scalar_small(_lib.SCALAR_TYCHE_INIT, (seed, stream_counter & MASK32), 4))


def tyche_next(state) -> tuple[int, tuple[int, int, int, int]]:
    state = tyche_mix(state)
    return state[1], state


# ---------------------------------------------------------------------------
# Engine
# ---------------------------------------------------------------------------

_PF_MIN, _PF_MAX = 64, 1 << 16


class Generator:
    """Deterministic 32-bit word stream named by (algorithm, seed, counter).

    Same contract as the reference engine (generators.py:227-395): `next_u32`
    draws one word, `words(n)` draws n in bulk and leaves the same state,
    `state_bytes`/`from_state_bytes` round-trip the 18-byte state.

    Scalar draws are served from a small host-side window of words prefetched
    from the GPU at the current stream position (the stream is a pure function
    of position, so prefetching is invisible to callers); bulk draws write
    straight into device memory.
    """

    MIN = 0
    MAX = MASK32

    __slots__ = ("algorithm", "seed", "stream_counter", "_block_ctr", "_cache_pos", "_key",
                 "_ty_state", "_ty_base", "_ty_pending", "_ty_win", "_pf", "_pf_pos", "_pf_n")

    def __init__(self, algorithm: Algorithm, seed: int, stream_counter: int):
        self.algorithm = as_algorithm(algorithm)
        self.seed = seed & MASK64
        self.stream_counter = stream_counter & MASK32
        if self.algorithm is Algorithm.SQUARES:
            self.seed &= MASK32  # generators.py:256-257
        self._block_ctr = 0
        self._cache_pos = 0
        self._key = self._derive_key()
        # Tyche: state after the last word handed to the window (_ty_state), the
        # state at the start of the window (_ty_base) and the words not yet served.
        self._ty_state = None
        self._ty_base = None
        self._ty_pending = None
        self._ty_win = 0
        # counter algorithms: prefetch window of words starting at word position _pf_pos
        self._pf = None
        self._pf_pos = 0
        self._pf_n = _PF_MIN

    def _derive_key(self):
        if self.algorithm is Algorithm.PHILOX:
            return (self.seed & MASK32, (self.seed >> 32) & MASK32)
        if self.algorithm is Algorithm.THREEFRY:
            return (self.seed & MASK32, (self.seed >> 32) & MASK32, self.stream_counter, 0)
        return None  # Squares key is expanded on the device (squares_key below)

    @property
    def stream_id(self) -> StreamId:
        return StreamId(self.seed, self.stream_counter)

    @property
    def words_per_block(self) -> int:
        return 4 if self.algorithm in (Algorithm.PHILOX, Algorithm.THREEFRY) else 1

    # ----- position bookkeeping (generators.py:285-312) -----
    def _word_pos(self) -> int:
        """Absolute word position (mod the stream period) of the next word."""
        if self.words_per_block == 4:
            blk = (self._block_ctr - (1 if self._cache_pos else 0)) & MASK32
            return blk * 4 + self._cache_pos
        return self._block_ctr

    def _advance(self, n: int) -> None:
        """Advance the logical state by n words exactly as n x next_u32 would."""
        if n <= 0:
            return
        if self.words_per_block == 4:
            pos = self._word_pos() + n
            self._cache_pos = pos & 3
            self._block_ctr = ((pos + 3) >> 2) & MASK32
        else:
            self._block_ctr = (self._block_ctr + n) & MASK32

    @property
    def _cache(self):
        """The partially served block (generators.py:306-311), computed on demand."""
        if self.words_per_block != 4 or self._cache_pos == 0:
            return None
        blk = (self._block_ctr - 1) & MASK32
        if self.algorithm is Algorithm.PHILOX:
            return philox_block(self._key, (self.stream_counter, blk, 0, 0))
        return threefry_block(self._key, (blk, 0, 0, 0))

    # ----- Tyche serial state -----
    def _tyche_end_state(self):
        """State after every word already served or pending in the window."""
        if self._ty_state is None:
            self._ty_state = tyche_init(self.seed, self.stream_counter)
            self._ty_base = self._ty_state
            self._ty_pending = np.empty(0, np.uint32)
            self._ty_win = 0
        return self._ty_state

    @property
    def _tyche_state(self):
        """Logical Tyche state at the current position (generators.py:262-265)."""
        if self.algorithm is not Algorithm.TYCHE:
            return None
        end = self._tyche_end_state()
        if self._ty_pending.size == 0:
            return end
        from . import bulk

        return bulk.tyche_advance_state(self._ty_base, self._ty_win - self._ty_pending.size)

    # ----- scalar draws -----
    def next_u32(self) -> int:
        """Next 32-bit word of the stream."""
        if self.algorithm is Algorithm.TYCHE:
            if self._ty_state is None or self._ty_pending.size == 0:
                from . import _lib

                n = self._pf_n
                self._pf_n = min(self._pf_n * 2, _PF_MAX)
                if self._ty_state is None:  # fresh stream: init + first window in one round trip
                    r = _lib.scalar(_lib.SCALAR_TYCHE_SEED_WORDS, [self.seed, self.stream_counter], n + 8)
                    self._ty_base = tuple(r[:4].tolist())
                    self._ty_pending, self._ty_state = r[4:4 + n], tuple(r[4 + n:].tolist())
                else:
                    self._ty_base = self._ty_state
                    r = _lib.scalar(_lib.SCALAR_TYCHE_WORDS, self._ty_state, n + 4)
                    self._ty_pending, self._ty_state = r[:n], tuple(r[n:].tolist())
                self._ty_win = n
            w = int(self._ty_pending[0])
            self._ty_pending = self._ty_pending[1:]
            self._block_ctr = (self._block_ctr + 1) & MASK32
            return w
        pos = self._word_pos()
        period = 1 << 34 if self.words_per_block == 4 else 1 << 32
        if self._pf is None or not (0 <= (pos - self._pf_pos) % period < self._pf.size):
            self._refill(pos)
        w = int(self._pf[(pos - self._pf_pos) % period])
        self._advance(1)
        return w

    def _refill(self, pos: int) -> None:
        from . import _lib

        n = self._pf_n
        self._pf_n = min(self._pf_n * 2, _PF_MAX)
        self._pf = _lib.scalar(_lib.SCALAR_STREAM_WORDS, [int(self.algorithm), self.seed, self.stream_counter, pos], n)
        self._pf_pos = pos

    __call__ = next_u32

    def next_u64(self) -> int:
        """Two word draws recombined, low word first (generators.py:316-320)."""
        lo = self.next_u32()
        hi = self.next_u32()
        return (hi << 32) | lo

    def words(self, n: int, *, out=None, device=None):
        """Next n words (bulk.generator_words): a uint32 CUDA tensor by default,
        a numpy array with device="cpu", or written into `out`."""
        from . import bulk

        return bulk.generator_words(self, n, out=out, device=device)

    def copy(self) -> "Generator":
        g = type(self).__new__(type(self))
        for name in Generator.__slots__:
            setattr(g, name, getattr(self, name))
        return g

    def state_bytes(self) -> bytes:
        """18-byte little-endian state (generators.py:345-353)."""
        return STATE_STRUCT.pack(int(self.algorithm), self.seed, self.stream_counter, self._block_ctr,
                                 self._cache_pos)

    @classmethod
    def from_state_bytes(cls, data: bytes) -> "Generator":
        """generators.py:355-374"""
        tag, seed, stream_ctr, block_ctr, cache_pos = STATE_STRUCT.unpack(data)
        g = Generator(Algorithm(tag), seed, stream_ctr)
        if cls is not Generator:  # Philox.from_state_bytes(...) etc.: same engine, the subclass's type
            fixed = getattr(cls, "ALGORITHM", None)
            if fixed is not None and fixed is not g.algorithm:
                raise ValueError(f"state is for {g.algorithm.name.lower()}, not {fixed.name.lower()}")
            g.__class__ = cls
        if g.words_per_block == 1:
            if cache_pos != 0:
                raise ValueError("cache position must be 0 for single-word algorithms")
            if g.algorithm is Algorithm.TYCHE and block_ctr:
                from . import bulk

                g._ty_state = bulk.tyche_advance_state(tyche_init(g.seed, g.stream_counter), block_ctr)
                g._ty_base = g._ty_state
                g._ty_pending = np.empty(0, np.uint32)
                g._ty_win = 0
            g._block_ctr = block_ctr
            return g
        if cache_pos > 3:
            raise ValueError("cache position must be < 4")
        g._block_ctr = block_ctr
        g._cache_pos = cache_pos
        return g

    def __repr__(self) -> str:
        return (f"Generator({self.algorithm.name.lower()}, seed={self.seed:#x}, "
                f"stream_counter={self.stream_counter}, position={self._position()})")

    def _position(self) -> int:
        if self._cache_pos:
            return ((self._block_ctr - 1) & MASK32) * 4 + self._cache_pos
        return self._block_ctr * self.words_per_block


def make_generator(algorithm, seed: int, counter: int) -> Generator:
    """Engine positioned at the start of stream (seed, counter) (generators.py:398-406)."""
    return Generator(as_algorithm(algorithm), seed, counter)


class Philox(Generator):
    """Philox4x32-10 stream (seed, counter): the OpenRAND `Philox` generator class."""

    __slots__ = ()
    ALGORITHM = Algorithm.PHILOX

    def __init__(self, seed: int, counter: int = 0):
        super().__init__(Algorithm.PHILOX, seed, counter)


class Threefry(Generator):
    __slots__ = ()
    ALGORITHM = Algorithm.THREEFRY

    def __init__(self, seed: int, counter: int = 0):
        super().__init__(Algorithm.THREEFRY, seed, counter)


class Squares(Generator):
    __slots__ = ()
    ALGORITHM = Algorithm.SQUARES

    def __init__(self, seed: int, counter: int = 0):
        super().__init__(Algorithm.SQUARES, seed, counter)


class Tyche(Generator):
    __slots__ = ()
    ALGORITHM = Algorithm.TYCHE

    def __init__(self, seed: int, counter: int = 0):
        super().__init__(Algorithm.TYCHE, seed, counter)
