"""Dense univariate polynomials over a prime field (host-side container).

Mirrors the reference's DensePoly (/root/reference/pkg/src/modconv/poly.py:
26-82), the input/output type of poly_mul: an immutable (field, coeffs) pair
with every coefficient a canonical residue, trailing zeros allowed and
stripped by normalize().  The reference's classical multipliers
(mul_schoolbook / mul_karatsuba, poly.py:90-169) run on the GPU's
defining-sum kernel (mc_conv_direct); eval_poly is host-side Horner.
"""

from __future__ import annotations

from dataclasses import dataclass

from .field import FieldMismatchError, FourierPrime, as_field


class PolyTextError(ValueError):
    """Malformed polynomial text; `line` is the 1-based offending line
    (poly.py:14-19 of the reference)."""

    def __init__(self, message: str, line: int):
        super().__init__(f"line {line}: {message}")
        self.line = line


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
    def _trusted(cls, fp: FourierPrime, coeffs: tuple) -> "DensePoly":
        """Wrap coefficients already known to be canonical residues (engine
        outputs) without the per-coefficient range check."""
        obj = object.__new__(cls)
        object.__setattr__(obj, "field", fp)
        object.__setattr__(obj, "coeffs", coeffs)
        return obj

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


# ------------------------------------------------------------------ direct products
# The reference's quadratic and divide-and-conquer multipliers (poly.py:90-181)
# share one output contract -- the raw coefficient product, NOT normalized --
# which the GPU defining-sum kernel (mc_conv_direct) computes for any field
# and length.
KARATSUBA_THRESHOLD = 16  # poly.py:15 (a tuning knob there; accepted and validated here)


def schoolbook_raw(a, b, p: int) -> list[int]:
    """Coefficient product of two nonempty sequences mod p (poly.py:90-97)."""
    if len(a) == 0 or len(b) == 0:
        raise ValueError("inputs must be nonempty")
    from .convolve import lin_conv_def

    return lin_conv_def(list(a), list(b), p)


def mul_schoolbook(a, b) -> DensePoly:
    """Direct convolution product c_k = sum_{i+j=k} a_i b_j (poly.py:100-105)."""
    check_same_field(a, b)
    fp = as_field(a.field)
    if a.is_zero() or b.is_zero():
        return DensePoly.zero(fp)
    return DensePoly._trusted(fp, tuple(schoolbook_raw(a.coeffs, b.coeffs, fp.p)))


def mul_karatsuba(a, b, threshold: int = KARATSUBA_THRESHOLD) -> DensePoly:
    """Same output contract as mul_schoolbook, bit for bit (poly.py:156-169)."""
    check_same_field(a, b)
    if threshold < 1:
        raise ValueError("threshold must be >= 1")
    return mul_schoolbook(a, b)


def eval_poly(a, x):
    """Horner evaluation of a at the point x (poly.py:172-181)."""
    from .field import Felt

    if a.field.p != x.field.p:
        raise FieldMismatchError(f"mixed moduli {a.field.p} and {x.field.p}")
    p = a.field.p
    xv = x.value
    acc = 0
    for c in reversed(a.coeffs):
        acc = (acc * xv + c) % p
    return Felt(acc, as_field(a.field))


# ------------------------------------------------------------------ text format
# Interchange format of the reference CLI (poly.py:184-223): three lines --
# the modulus, the coefficient count, the space-separated residues.

def poly_to_text(a) -> str:
    return f"{a.field.p}\n{len(a.coeffs)}\n{' '.join(str(int(c)) for c in a.coeffs)}\n"


def _parse_int(token: str, what: str, line: int) -> int:
    try:
        return int(token)
    except ValueError:
        raise PolyTextError(f"bad {what} {token!r}", line) from None


def poly_from_text(text: str, field=None) -> DensePoly:
    """Parse the three-line format; errors carry the offending line."""
    head = text.splitlines()
    if len(head) < 3:
        raise PolyTextError("expected 3 lines: modulus, count, coefficients", len(head) + 1)
    modulus_line, count_line, coeff_line = head[0], head[1], head[2]
    p = _parse_int(modulus_line, "modulus", 1)
    if field is not None and field.p == p:
        fp = as_field(field)
    else:
        try:
            fp = as_field(p)
        except ValueError as exc:
            raise PolyTextError(str(exc), 1) from None
    count = _parse_int(count_line, "coefficient count", 2)
    if count < 0:
        raise PolyTextError(f"negative coefficient count {count}", 2)
    values = [_parse_int(tok, "coefficient", 3) for tok in coeff_line.split()]
    if len(values) != count:
        raise PolyTextError(f"expected {count} coefficients, found {len(values)}", 3)
    bad = next((v for v in values if not 0 <= v < p), None)
    if bad is not None:
        raise PolyTextError(f"coefficient {bad} not a canonical residue mod {p}", 3)
    return DensePoly(fp, tuple(values))
