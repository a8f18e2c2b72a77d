"""Degenerate circuits with closed-form amplitudes (shared by the oracle pins and the GPU
parity tests): a single qubit, a product state (no two-qubit gate), no gates at all, and
two disconnected components (the contraction tree then multiplies scalars / outer
products, Eq. (3) with no shared index)."""
import numpy as np

from tn_inputs import Circuit
from tn_inputs.circuits import haar_unitary


def degenerate_circuits():
    """[(circuit, amplitude(x) closed form)]; <x|C|0> with x_q the bit of qubit q and a
    two-qubit gate's basis |x_a x_b> (x_a the high bit, tn.h)."""
    rng = np.random.default_rng(77)
    out = []
    U = haar_unitary(rng, 2)
    c = Circuit(1, np.zeros((1, 2)), name="one_qubit")
    c.add((0,), U)
    out.append((c, lambda x, U=U: U[x[0], 0]))

    Us = [[haar_unitary(rng, 2) for _ in range(2)] for _ in range(3)]
    c = Circuit(3, np.array([[0.0, 0.0], [1.0, 0.0], [2.0, 0.0]]), name="product3")
    for q in range(3):
        for V in Us[q]:
            c.add((q,), V)
    out.append((c, lambda x, Us=Us: np.prod([(Us[q][1] @ Us[q][0])[x[q], 0] for q in range(3)])))

    c = Circuit(2, np.array([[0.0, 0.0], [1.0, 0.0]]), name="no_gates")
    out.append((c, lambda x: 1.0 + 0j if not np.any(x) else 0j))

    U4, V2, V3 = haar_unitary(rng, 4), haar_unitary(rng, 2), haar_unitary(rng, 2)
    c = Circuit(4, np.array([[0.0, 0.0], [1.0, 0.0], [5.0, 0.0], [9.0, 0.0]]), name="split4")
    c.add((0, 1), U4)
    c.add((2,), V2)
    c.add((3,), V3)
    out.append((c, lambda x, U4=U4, V2=V2, V3=V3: U4[2 * x[0] + x[1], 0] * V2[x[2], 0] * V3[x[3], 0]))
    return out


def all_bitstrings(n):
    return np.array([[(i >> (n - 1 - q)) & 1 for q in range(n)] for i in range(1 << n)], dtype=np.uint8)
