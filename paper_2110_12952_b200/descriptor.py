"""NBB fractal descriptors: host-side mirror of proj/include/nbb/descriptor.hpp.

FractalDescriptor(name, k, s, replicas): k replicas on an s x s sub-box grid;
the order of ``replicas`` defines replica IDs 0..k-1 (descriptor.hpp:21-36).
Validation follows FractalDescriptor::validate (proj/src/descriptor.cpp:12-44),
the three built-ins follow builtin_descriptor (descriptor.cpp:53-64) and the
``key=value`` file format follows parse_descriptor (descriptor.cpp:110-149).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Tuple

from .errors import ParseError, OutOfDomain, CapacityError

INT64_MAX = (1 << 63) - 1


@dataclass
class FractalDescriptor:
    name: str = ""
    replica_count: int = 0  # k
    growth: int = 0  # s
    replicas: List[Tuple[int, int]] = field(default_factory=list)

    @property
    def k(self) -> int:
        return self.replica_count

    @property
    def s(self) -> int:
        return self.growth

    def validate(self) -> None:
        """descriptor.cpp:12-44"""
        n, k, s = self.name, self.replica_count, self.growth
        if k < 1:
            raise ParseError(f"descriptor '{n}': k must be >= 1, got {k}")
        if s < 2:
            raise ParseError(f"descriptor '{n}': invalid growth factor s={s} (s >= 2 required)")
        if k > s * s:
            raise ParseError(f"descriptor '{n}': k={k} exceeds s*s={s * s}")
        if len(self.replicas) != k:
            raise ParseError(f"descriptor '{n}': k={k} but {len(self.replicas)} replica positions listed")
        for i, (gx, gy) in enumerate(self.replicas):
            if gx < 0 or gy < 0 or gx >= s or gy >= s:
                raise ParseError(f"descriptor '{n}': replica {i} position ({gx},{gy}) outside the "
                                 f"{s}x{s} grid")
            for j in range(i + 1, len(self.replicas)):
                if self.replicas[j] == (gx, gy):
                    raise ParseError(f"descriptor '{n}': duplicate replica position ({gx},{gy})")

    def replica_index(self, gx: int, gy: int) -> int:
        """descriptor.cpp:46-51"""
        for i, p in enumerate(self.replicas):
            if p == (gx, gy):
                return i
        return -1

    def flat_replicas(self) -> List[int]:
        return [v for xy in self.replicas for v in xy]


def builtin_descriptor(name: str) -> FractalDescriptor:
    """descriptor.cpp:53-64"""
    if name == "sierpinski-triangle":
        return FractalDescriptor("sierpinski-triangle", 3, 2, [(0, 0), (1, 0), (0, 1)])
    if name == "sierpinski-carpet":
        return FractalDescriptor("sierpinski-carpet", 8, 3,
                                 [(0, 0), (1, 0), (2, 0), (0, 1), (2, 1), (0, 2), (1, 2), (2, 2)])
    if name == "vicsek":
        return FractalDescriptor("vicsek", 5, 3, [(1, 0), (0, 1), (1, 1), (2, 1), (1, 2)])
    raise ParseError(f"unknown fractal name '{name}' (builtins: sierpinski-triangle, "
                     "sierpinski-carpet, vicsek; use @file for a descriptor file)")


def _parse_int(tok: str, what: str) -> int:
    tok = tok.strip()
    # std::from_chars(int): optional '-', decimal digits, whole token consumed
    body = tok[1:] if tok.startswith("-") else tok
    if not body or not body.isdigit() or not body.isascii():
        raise ParseError(f"malformed {what} value '{tok}'")
    v = int(tok)
    if v < -(1 << 31) or v > (1 << 31) - 1:
        raise ParseError(f"malformed {what} value '{tok}'")
    return v


def _parse_replicas(text: str) -> List[Tuple[int, int]]:
    out = []
    for pair in text.split(";"):
        pair = pair.strip()
        if not pair:
            continue
        if "," not in pair:
            raise ParseError(f"malformed replica pair '{pair}' (expected gx,gy)")
        a, b = pair.split(",", 1)
        out.append((_parse_int(a, "replica gx"), _parse_int(b, "replica gy")))
    return out


def parse_descriptor(text: str) -> FractalDescriptor:
    """descriptor.cpp:110-149"""
    d = FractalDescriptor()
    seen = set()
    for raw in text.split("\n"):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        if "=" not in line:
            raise ParseError(f"malformed descriptor line '{line}' (expected key=value)")
        key, value = line.split("=", 1)
        key, value = key.strip(), value.strip()
        if key == "name":
            d.name = value
        elif key == "k":
            d.replica_count = _parse_int(value, "k")
        elif key == "s":
            d.growth = _parse_int(value, "s")
        elif key == "replicas":
            d.replicas = _parse_replicas(value)
        else:
            raise ParseError(f"unknown descriptor key '{key}'")
        seen.add(key)
    if not {"name", "k", "s", "replicas"} <= seen:
        raise ParseError("descriptor is missing required keys (need name, k, s, replicas)")
    d.validate()
    return d


def load_descriptor(spec: str) -> FractalDescriptor:
    """descriptor.cpp:151-162: a built-in name or '@path'."""
    if spec.startswith("@"):
        path = spec[1:]
        try:
            with open(path, "r") as fh:
                text = fh.read()
        except OSError:
            raise ParseError(f"cannot open descriptor file '{path}'") from None
        return parse_descriptor(text)
    return builtin_descriptor(spec)


# ----------------------------------------------------------------------------
# geometry (proj/src/geometry.cpp) -- the sizes that drive device allocation
# ----------------------------------------------------------------------------
def ipow_checked(base: int, exp: int) -> int:
    """geometry.cpp:10-21"""
    if base < 0 or exp < 0:
        raise CapacityError("ipow_checked: negative base or exponent")
    r = 1
    for _ in range(exp):
        if base != 0 and r > INT64_MAX // base:
            raise CapacityError(f"integer overflow computing {base}^{exp}")
        r *= base
    return r


def side_length(d: FractalDescriptor, level: int) -> int:
    if level < 0:
        raise OutOfDomain("scale level must be >= 0")
    return ipow_checked(d.growth, level)


def cell_count(d: FractalDescriptor, level: int) -> int:
    if level < 0:
        raise OutOfDomain("scale level must be >= 0")
    return ipow_checked(d.replica_count, level)


def compact_dims(d: FractalDescriptor, level: int) -> Tuple[int, int]:
    """maps.cpp:36-43"""
    if level < 0:
        raise OutOfDomain("scale level must be >= 0")
    return ipow_checked(d.replica_count, (level + 1) // 2), ipow_checked(d.replica_count, level // 2)


def unfold_stride(k: int, mu: int) -> Tuple[int, int]:
    """maps.cpp:28-34"""
    if mu < 0:
        raise OutOfDomain("level index must be >= 0")
    p = ipow_checked(k, mu // 2)
    return (p, 0) if mu % 2 == 0 else (0, p)


def hausdorff_dimension(d: FractalDescriptor) -> float:
    return math.log(d.replica_count) / math.log(d.growth)
