"""Dense univariate polynomials over a prime field (host-side container).

Mirrors the reference's DensePoly (/root/reference/pkg/src/modconv/poly.py:
26-82), the input/output type of poly_mul: an immutable (field, coeffs) pair
with every coefficient a canonical residue, trailing zeros allowed and
stripped by normalize().  The classical O(n^2) multipliers of the reference
are test oracles and live under oracle/, not here.
"""

from __future__ import annotations

from dataclasses import dataclass

from .field import FieldMismatchError, FourierPrime, as_field


@dataclass(frozen=True, slots=True)
class DensePoly:
    field: FourierPrime
    coeffs: tuple

    def __post_init__(self) -> None:
        if not isinstance(self.coeffs, tuple):
            object.__setattr__(self, "coeffs", tuple(self.coeffs))
        p = self.field.p
        for c in self.coeffs:
            if not 0 <= c < p:
                raise ValueError(f"coefficient {c} out of range for p={p}")

    @classmethod
    def from_ints(cls, field, values) -> "DensePoly":
        """Reduce arbitrary integers mod p (poly.py:46-49)."""
        fp = as_field(field)
        p = fp.p
        return cls(fp, tuple(int(v) % p for v in values))

    @classmethod
    def zero(cls, field) -> "DensePoly":
        return cls(as_field(field), ())

    @classmethod
    def one(cls, field) -> "DensePoly":
        return cls(as_field(field), (1,))

    def __len__(self) -> int:
        return len(self.coeffs)

    def is_zero(self) -> bool:
        return not any(self.coeffs)

    def degree(self):
        for i in range(len(self.coeffs) - 1, -1, -1):
            if self.coeffs[i]:
                return i
        return None

    def normalize(self) -> "DensePoly":
        """Drop trailing zeros; idempotent (poly.py:72-79)."""
        d = self.degree()
        if d is None:
            return DensePoly(self.field, ())
        if d == len(self.coeffs) - 1:
            return self
        return DensePoly(self.field, self.coeffs[: d + 1])

    def __repr__(self) -> str:
        return f"DensePoly(p={self.field.p}, coeffs={self.coeffs})"


def check_same_field(a, b) -> None:
    if a.field.p != b.field.p:
        raise FieldMismatchError(f"mixed moduli {a.field.p} and {b.field.p}")
