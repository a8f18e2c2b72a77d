"""Brute-force state-vector simulation (TEST INFRASTRUCTURE -- oracle).

Independent of the tensor-network path: applies every gate of the circuit to the
dense 2^N state |0...0> and reads <x|C|0> ("explicit time
evolution").  Used to pin oracle.network + oracle.contract on small circuits.
"""
from __future__ import annotations

import numpy as np


def statevector(circ) -> np.ndarray:
    n = circ.n
    psi = np.zeros((2,) * n, dtype=np.complex128)
    psi[(0,) * n] = 1.0
    for qs, U in circ.gates:
        if len(qs) == 1:
            (q,) = qs
            psi = np.moveaxis(np.tensordot(U, psi, axes=([1], [q])), 0, q)
        else:
            a, b = qs
            G = U.reshape(2, 2, 2, 2)          # [a_out, b_out, a_in, b_in]
            psi = np.tensordot(G, psi, axes=([2, 3], [a, b]))
            psi = np.moveaxis(psi, [0, 1], [a, b])
    return psi


def amplitude(circ, bits) -> complex:
    psi = statevector(circ)
    return complex(psi[tuple(int(b) for b in bits)])
