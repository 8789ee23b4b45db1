"""Minimal Pauli-sum operator for ``run(..., hamiltonian=...)``.

The reference's PauliHamiltonian (nucsim/hamiltonian.py:59-176) belongs to
its physics front end, which is out of scope here.  The engine only needs
the three members ``n_qubits``, ``sorted_terms()`` and ``is_hermitian()``,
so any object providing them (including the reference's own class) is
accepted; this class provides them for standalone use.  Letter strings are
qubit-0-first (hamiltonian.py:1-6).
"""

from __future__ import annotations

_LETTERS = frozenset("IXYZ")


class PauliHamiltonian:
    def __init__(self, n_qubits: int, terms: dict[str, complex] | None = None):
        if n_qubits < 1:
            raise ValueError("need at least one qubit")
        self.n_qubits = n_qubits
        self.terms: dict[str, complex] = {}
        for letters, coeff in (terms or {}).items():
            if len(letters) != n_qubits or set(letters) - _LETTERS:
                raise ValueError(f"bad Pauli string {letters!r} for {n_qubits} qubits")
            if abs(coeff) > 1e-14:
                self.terms[letters] = complex(coeff)

    def sorted_terms(self) -> list[tuple[str, complex]]:
        return sorted(self.terms.items())

    def is_hermitian(self, atol: float = 1e-9) -> bool:
        return all(abs(c.imag) <= atol for c in self.terms.values())

    def __len__(self) -> int:
        return len(self.terms)


def term_masks(letters: str) -> tuple[int, int, int]:
    """(x-mask, z-mask, #Y) of a Pauli word; P psi[j] = (-i)^#Y
    (-1)^popcount(j & z) psi[j ^ x] (the action of hamiltonian.py:179-194)."""
    x = z = ny = 0
    for q, c in enumerate(letters):
        if c in "XY":
            x |= 1 << q
        if c in "ZY":
            z |= 1 << q
        ny += c == "Y"
    return x, z, ny
