import sys, os; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, test_gpu as T, paper_2208_01498_b200 as tb
from tn_inputs import lattice_cz, random_bitstrings
from oracle.network import build_network
from oracle.ssa import find_order
from oracle.contract import contract_tree
c = lattice_cz(6, 6, 12, 8)
on = build_network(c); st, _ = find_order(on, seed=0)
cn = tb.Network.from_circuit(c); co = tb.Order(cn, seed=0)
plan = tb.Plan(cn, co, dtype=tb.TN_C64)
steps = plan.steps()
print("tc steps", [tuple(r[1:5]) for r in steps if r[0] == tb.TN_PATH_TC])
x = np.zeros(c.n, np.uint8)
print(os.environ.get("TN_PACK_CAP_LOG2"), os.environ.get("TN_ROW_SLABS"), os.environ.get("TN_GEMM_PAIR"), plan.contract(x), contract_tree(on, st, x))
