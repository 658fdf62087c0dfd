"""Problem instances (mirror of gsetbench.instances, instances.py:19-239).

Toroidal instances keep their +-1 couplings as one int8 array
``w[2x] = right edge of site x, w[2x+1] = down edge`` -- the emission order of
generate_torus (instances.py:211-223) -- and build the reference's tuple views
(edges, adjacency) only when asked, so the 2000x2000 configuration costs 8 MB
instead of ~6 GB of Python tuples.  Device copies are generated on the GPU
(gsb_torus_weights) and cached per device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class GsetFormatError(ValueError):
    """Raised when instance text or edge data violates the format."""


class ProblemInstance:
    """Immutable weighted graph, vertices 1..n, edges canonical (u, v, w), u < v.

    Equality compares structure only (instances.py:19-27).
    """

    __slots__ = ("n", "name", "_edges", "_torus", "_w", "_eu", "_ev", "_ew", "_adj", "_dev",
                 "_frozen")

    def __init__(self, n: int, edges=(), name: str = "", *, _torus=None, _w=None):
        s = object.__setattr__
        s(self, "n", int(n))
        s(self, "name", name)
        s(self, "_torus", _torus)
        s(self, "_w", _w)
        s(self, "_eu", None)
        s(self, "_ev", None)
        s(self, "_ew", None)
        s(self, "_adj", None)
        s(self, "_dev", {})
        if self.n < 1:
            raise GsetFormatError(f"vertex count must be positive, got {self.n}")
        if _torus is None:
            edges = tuple((int(u), int(v), int(w)) for u, v, w in edges)
            arr = np.asarray(edges, dtype=np.int64).reshape(-1, 3)
            bad = np.nonzero(~((arr[:, 0] >= 1) & (arr[:, 0] < arr[:, 1]) & (arr[:, 1] <= self.n)))[0]
            if bad.size:
                i = int(bad[0])
                u, v, _ = edges[i]
                raise GsetFormatError(
                    f"edge {i + 1}: endpoints ({u}, {v}) not canonical for n={self.n}")
            s(self, "_edges", edges)
            s(self, "_eu", arr[:, 0] - 1)
            s(self, "_ev", arr[:, 1] - 1)
            s(self, "_ew", arr[:, 2].copy())
        else:
            s(self, "_edges", None)
        s(self, "_frozen", True)

    def __setattr__(self, key, value):
        raise AttributeError("ProblemInstance is immutable")

    # ---- reference surface -------------------------------------------------
    @classmethod
    def from_edges(cls, n: int, edges, name: str = "") -> "ProblemInstance":
        """instances.py:64-94: normalise to u < v, reject loops/range/duplicates."""
        if n < 1:
            raise GsetFormatError(f"vertex count must be positive, got {n}")
        seen: set[tuple[int, int]] = set()
        canonical = []
        for i, (u, v, w) in enumerate(edges):
            if u == v:
                raise GsetFormatError(f"edge {i + 1}: self-loop at vertex {u}")
            if not (1 <= u <= n) or not (1 <= v <= n):
                raise GsetFormatError(f"edge {i + 1}: endpoint out of range 1..{n}: ({u}, {v})")
            if u > v:
                u, v = v, u
            if (u, v) in seen:
                raise GsetFormatError(f"edge {i + 1}: duplicate edge ({u}, {v})")
            seen.add((u, v))
            canonical.append((u, v, int(w)))
        return cls(n=n, edges=tuple(canonical), name=name)

    @property
    def edges(self) -> tuple[tuple[int, int, int], ...]:
        if self._edges is None:
            self._materialise_torus_edges()
        return self._edges

    @property
    def m(self) -> int:
        if self._torus is not None:
            return 2 * self.n
        return len(self._edges)

    @property
    def adjacency(self):
        """Neighbour lists indexed by vertex id; entry 0 unused (instances.py:100-103)."""
        if self._adj is None:
            adj = [[] for _ in range(self.n + 1)]
            for u, v, w in self.edges:
                adj[u].append((v, w))
                adj[v].append((u, w))
            object.__setattr__(self, "_adj", tuple(tuple(x) for x in adj))
        return self._adj

    def total_weight(self) -> int:
        if self._torus is not None:
            return int(self._w.astype(np.int64).sum())
        return int(self._ew.sum())

    def __eq__(self, other):
        if not isinstance(other, ProblemInstance):
            return NotImplemented
        if self._torus is not None and other._torus is not None:
            return (self._torus.rows, self._torus.cols) == (other._torus.rows, other._torus.cols) \
                and np.array_equal(self._w, other._w)
        return self.n == other.n and self.edges == other.edges

    def __hash__(self):
        return hash((self.n, self.edges))

    def __repr__(self):
        return f"ProblemInstance(n={self.n}, m={self.m}, name={self.name!r})"

    # ---- engine-facing -----------------------------------------------------
    @property
    def torus(self) -> "TorusSpec | None":
        return self._torus

    @property
    def torus_weights(self) -> np.ndarray:
        """int8 [2n] couplings in emission order (torus instances only)."""
        if self._torus is None:
            raise ValueError("not a torus instance")
        return self._w

    def edge_arrays(self):
        """0-based int64 (eu, ev, ew) as evaluate.py uses them (instances.py:43-59)."""
        if self._eu is None:
            self._materialise_torus_edges()
        return self._eu, self._ev, self._ew

    def _materialise_torus_edges(self):
        spec = self._torus
        rows, cols = spec.rows, spec.cols
        r, c = np.meshgrid(np.arange(rows), np.arange(cols), indexing="ij")
        vid = (r * cols + c).ravel()
        right = (r * cols + (c + 1) % cols).ravel()
        down = (((r + 1) % rows) * cols + c).ravel()
        a = np.stack([vid, vid], axis=1).ravel()
        b = np.stack([right, down], axis=1).ravel()
        eu = np.minimum(a, b).astype(np.int64)
        ev = np.maximum(a, b).astype(np.int64)
        ew = self._w.astype(np.int64)
        object.__setattr__(self, "_eu", eu)
        object.__setattr__(self, "_ev", ev)
        object.__setattr__(self, "_ew", ew)
        object.__setattr__(self, "_edges", tuple(
            (int(u) + 1, int(v) + 1, int(w)) for u, v, w in zip(eu, ev, ew)))

    def device_weights(self, device):
        """Cached device int8 couplings, generated on the GPU (gsb_torus_weights)."""
        import torch

        from paper_2505_18508_b200 import _lib

        dev = torch.device(device)
        key = ("w", dev.index)
        t = self._dev.get(key)
        if t is None:
            _lib.require_cuda()
            t = torch.empty(2 * self.n, dtype=torch.int8, device=dev)
            with torch.cuda.device(dev):
                stream = torch.cuda.current_stream(dev).cuda_stream
                _lib.check(_lib.lib().gsb_torus_weights(self._torus.rows, self._torus.cols,
                                                        self._torus.seed, t.data_ptr(), stream))
            self._dev[key] = t
        return t

    def device_edges(self, device):
        """Cached device int32 (eu, ev, ew) for the general-graph engine."""
        import torch

        dev = torch.device(device)
        key = ("e", dev.index)
        t = self._dev.get(key)
        if t is None:
            eu, ev, ew = self.edge_arrays()
            if ew.size and (ew.max() >= 2**31 or ew.min() < -2**31):
                raise ValueError("edge weights must fit in int32")
            t = tuple(torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(dev)
                      for a in (eu, ev, ew))
            self._dev[key] = t
        return t


def _gset_error(text: str) -> None:
    """Token-by-token pass that names what is wrong with a Gset text and where
    (the messages of instances.py:117-158); only runs after the fast path failed."""
    tokens = [(no, tok) for no, line in enumerate(text.splitlines(), start=1)
              for tok in line.split("#", 1)[0].split()]
    pos = 0

    def take(what):
        nonlocal pos
        if pos >= len(tokens):
            raise GsetFormatError(f"unexpected end of input while reading {what}")
        no, tok = tokens[pos]
        pos += 1
        try:
            return int(tok)
        except ValueError:
            raise GsetFormatError(f"line {no}: expected integer {what}, got {tok!r}") from None

    n, m = take("vertex count"), take("edge count")
    if n < 1:
        raise GsetFormatError(f"vertex count must be positive, got {n}")
    if m < 0:
        raise GsetFormatError(f"edge count must be non-negative, got {m}")
    for i in range(m):
        take(f"edge {i + 1} endpoint")
        take(f"edge {i + 1} endpoint")
        take(f"edge {i + 1} weight")
    if pos < len(tokens):
        raise GsetFormatError(f"line {tokens[pos][0]}: trailing token {tokens[pos][1]!r} after "
                              f"{m} edges")
    raise GsetFormatError("malformed Gset text")


def parse_gset(text: str, name: str = "") -> ProblemInstance:
    """Gset text -> instance (instances.py:117-158): ``n m`` then m triples
    ``u v w``, any whitespace layout, ``#`` comments.  All tokens are converted
    in one numpy call (an 8M-edge file parses in seconds, not minutes); the
    token loop that reports line numbers runs only for malformed input."""
    body = text if "#" not in text else "\n".join(ln.split("#", 1)[0] for ln in text.splitlines())
    try:
        vals = np.array(body.split(), dtype=np.int64)
    except (ValueError, OverflowError):
        vals = None
    if (vals is None or vals.size < 2 or vals[0] < 1 or vals[1] < 0
            or vals.size != 2 + 3 * int(vals[1])):
        _gset_error(text)
    n, m = int(vals[0]), int(vals[1])
    return ProblemInstance.from_edges(n, map(tuple, vals[2:].reshape(m, 3).tolist()), name=name)


@dataclass(frozen=True)
class TorusSpec:
    """instances.py:176-200."""

    rows: int
    cols: int
    seed: int

    def __post_init__(self) -> None:
        if self.rows < 3 or self.cols < 3:
            raise ValueError(f"torus must be at least 3x3, got {self.rows}x{self.cols}")
        if not (0 <= self.seed < 2**64):
            raise ValueError(f"seed must fit in 64 bits, got {self.seed}")

    @property
    def name(self) -> str:
        return f"torus:{self.rows}x{self.cols}:{self.seed}"


def torus_weights_host(spec: TorusSpec) -> np.ndarray:
    """default_rng(seed).integers(0, 2, 2n) * 2 - 1 (instances.py:221-222) as int8."""
    n = spec.rows * spec.cols
    b = np.random.default_rng(spec.seed).integers(0, 2, size=2 * n)
    return (b * 2 - 1).astype(np.int8)


def generate_torus(spec: TorusSpec) -> ProblemInstance:
    """instances.py:203-224; same weights, lazily materialised tuple views."""
    w = torus_weights_host(spec)
    w.setflags(write=False)
    return ProblemInstance(spec.rows * spec.cols, name=spec.name, _torus=spec, _w=w)


def parse_torus_name(name: str) -> TorusSpec:
    """instances.py:227-239."""
    parts = name.split(":")
    if len(parts) != 3 or parts[0] != "torus":
        raise ValueError(f"not a torus name: {name!r}")
    dims = parts[1].split("x")
    if len(dims) != 2:
        raise ValueError(f"bad torus dimensions in {name!r}")
    try:
        rows, cols, seed = int(dims[0]), int(dims[1]), int(parts[2])
    except ValueError:
        raise ValueError(f"bad torus name {name!r}") from None
    return TorusSpec(rows=rows, cols=cols, seed=seed)
