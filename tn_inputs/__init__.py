"""Seeded synthetic inputs shared by the oracle (oracle/) and the product path.

This package holds NO arithmetic of the method: it never builds a tensor network,
orders or contracts anything.  It only produces problem inputs -- circuit
descriptions (qubit positions + time-ordered gate lists with their matrices) and
output bitstrings -- for the circuit families of BASELINE.json's configs.
"""
from .circuits import (Circuit, lattice_cz, sycamore, iqp, random3d, inverse_circuit,
                       concat, random_bitstrings, config_circuit, CONFIGS)

__all__ = ["Circuit", "lattice_cz", "sycamore", "iqp", "random3d", "inverse_circuit",
           "concat", "random_bitstrings", "config_circuit", "CONFIGS"]
