"""Per-launch device times of one step of a config (TN_PROFILE_DUMP): python scripts/prof_dump.py <config> <slice_log2> [min_ms]"""
import os, sys
os.environ.setdefault("TN_PROFILE_DUMP", sys.argv[3] if len(sys.argv) > 3 else "0.5")
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2208_01498_b200 as tb
from tn_inputs import config_circuit, random_bitstrings, CONFIGS
ci, tgt = int(sys.argv[1]), int(sys.argv[2])
c = config_circuit(ci)
net = tb.Network.from_circuit(c, diag_hyper=(ci == 3))
plan = tb.Plan(net, tb.Order(net, seed=0, n_seeds=int(os.environ.get("TN_SEEDS", "256")) if tgt else 4, max_log2_size=tgt), dtype=tb.TN_C64 if CONFIGS[ci]["dtype"] == "c64" else tb.TN_C128)
bits = torch.from_numpy(random_bitstrings(c.n, 1, 1)[0]).cuda()
amp = torch.zeros(1, dtype=torch.complex128, device="cuda")
plan.contract_profiled(bits.data_ptr(), 0, 1, amp.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("-- second run --", file=sys.stderr)
p = plan.contract_profiled(bits.data_ptr(), 1 % plan.info()["n_slices"], 1 % plan.info()["n_slices"] + 1, amp.data_ptr(), torch.cuda.current_stream().cuda_stream)
print(p)
