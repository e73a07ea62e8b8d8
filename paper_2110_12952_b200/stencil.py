"""Rule / neighbourhood / backend vocabulary: mirror of proj/include/nbb/stencil.hpp.

StencilRule.parse follows proj/src/stencil.cpp:11-41 (B<digits>/S<digits>, digits
0..8, either set may be empty, case-insensitive B/S); to_string follows
stencil.cpp:43-53; neighbor_offsets follows stencil.cpp:55-61; backend names
follow stencil.cpp:83-104 plus the two GPU backends this package adds.
"""
from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

from .errors import ParseError


class Neighborhood(Enum):
    VonNeumann = 0
    Moore = 1


@dataclass
class StencilRule:
    birth: int = 0
    survive: int = 0
    neighborhood: Neighborhood = Neighborhood.Moore

    def born_with(self, count: int) -> bool:
        return bool((self.birth >> count) & 1)

    def survives_with(self, count: int) -> bool:
        return bool((self.survive >> count) & 1)

    @staticmethod
    def parse(text: str, nb: Neighborhood = Neighborhood.Moore) -> "StencilRule":
        rule = StencilRule(0, 0, nb)
        pos = 0

        def expect(upper, lower):
            nonlocal pos
            if pos >= len(text) or text[pos] not in (upper, lower):
                raise ParseError(f"malformed rule '{text}' (expected B<digits>/S<digits>)")
            pos += 1

        def digits():
            nonlocal pos
            mask = 0
            while pos < len(text) and "0" <= text[pos] <= "9":
                c = ord(text[pos]) - ord("0")
                if c > 8:
                    raise ParseError(f"neighbor count {c} out of range [0,8] in rule '{text}'")
                mask |= 1 << c
                pos += 1
            return mask

        expect("B", "b")
        rule.birth = digits()
        expect("/", "/")
        expect("S", "s")
        rule.survive = digits()
        if pos != len(text):
            raise ParseError(f"trailing characters in rule '{text}'")
        return rule

    def to_string(self) -> str:
        return ("B" + "".join(str(c) for c in range(9) if self.born_with(c)) +
                "/S" + "".join(str(c) for c in range(9) if self.survives_with(c)))

    @property
    def moore(self) -> bool:
        return self.neighborhood == Neighborhood.Moore


def conway_rule() -> StencilRule:
    return StencilRule.parse("B3/S23")


_VN = [(1, 0), (-1, 0), (0, 1), (0, -1)]
_MOORE = _VN + [(1, 1), (1, -1), (-1, 1), (-1, -1)]


def neighbor_offsets(nb: Neighborhood):
    return list(_VN if nb == Neighborhood.VonNeumann else _MOORE)


class Backend(Enum):
    BoundingBox = "bb"
    CompactGrid = "lambda"
    Compact = "compact"
    GpuCompact = "gpu-compact"
    GpuBoundingBox = "gpu-bb"
    GpuLambda = "gpu-lambda"


def backend_name(b: Backend) -> str:
    return b.value


def parse_backend(name: str) -> Backend:
    for b in Backend:
        if b.value == name:
            return b
    raise ParseError(f"unknown backend '{name}' (expected bb, lambda, compact, gpu-compact, gpu-bb or gpu-lambda)")
