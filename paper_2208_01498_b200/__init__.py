"""B200-native tensor-network contraction of quantum-circuit amplitudes along
separator-based orders (arxiv 2208.01498, Wahl & Strelchuk).

Thin ctypes binding over the C ABI in include/tn.h (libtn_b200.so, built in-tree by
build.py).  Argument marshalling only: network construction and order search run
in the library's host C++, every contraction step runs in its sm_100a kernels.
There is no Python or CPU fallback: if the library is missing, importing the
binding's entry points raises.
"""
from ._lib import (lib, TnError, Network, Order, Plan, OrderParams, contract_pair, kernel_launches,
                   TN_C64, TN_C128, TN_PATH_AUTO, TN_PATH_SMALL, TN_PATH_TC, TN_PATH_SKINNY, TN_PATH_WIDE,
                   EXPORTED_SYMBOLS)

__all__ = ["lib", "TnError", "Network", "Order", "Plan", "OrderParams", "contract_pair", "kernel_launches",
           "TN_C64", "TN_C128", "TN_PATH_AUTO", "TN_PATH_SMALL", "TN_PATH_TC", "TN_PATH_SKINNY",
           "TN_PATH_WIDE", "EXPORTED_SYMBOLS"]
