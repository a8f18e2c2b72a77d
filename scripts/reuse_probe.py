"""Slice reuse on a config: arena, prologue share, time of the prologue and of a slice.
python scripts/reuse_probe.py <config> <target> [n_seeds]"""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2208_01498_b200 as tb
from tn_inputs import config_circuit, random_bitstrings, CONFIGS
ci, tgt = int(sys.argv[1]), int(sys.argv[2])
ns = int(sys.argv[3]) if len(sys.argv) > 3 else 256
c = config_circuit(ci)
net = tb.Network.from_circuit(c, diag_hyper=(ci == 3))
o = tb.Order(net, seed=0, n_seeds=ns, max_log2_size=tgt)
p = tb.Plan(net, o, dtype=tb.TN_C64 if CONFIGS[ci]["dtype"] == "c64" else tb.TN_C128)
i = p.info()
x = random_bitstrings(c.n, 1024, 1)[0]
contrib = p.contributing_slices(x)
print(f"config {ci} target 2^{tgt}: arena {i['arena_bytes'] / 1e9:.1f} GB, frontier {i['frontier_bytes'] / 1e9:.1f} GB, "
      f"prologue {i['flops_prologue'] / i['flops_per_slice']:.3f} of a slice, slice bits {i['slice_bits']}, contributing {contrib}", flush=True)
bits = torch.from_numpy(np.ascontiguousarray(x)).cuda()
amp = torch.zeros(1, dtype=torch.complex128, device='cuda')
st = torch.cuda.current_stream().cuda_stream
ids = p.contributing_slice_ids(x, 0, 3)
p.prepare(bits.data_ptr(), st)
p.contract_prepared(ids[0], ids[0] + 1, amp.data_ptr(), st)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
e[0].record(); p.prepare(bits.data_ptr(), st); e[1].record()
for s in ids[1:3]:
    p.contract_prepared(s, s + 1, amp.data_ptr(), st)
e[2].record(); torch.cuda.synchronize()
t_pro = e[0].elapsed_time(e[1]) / 1e3
t_sl = e[1].elapsed_time(e[2]) / 1e3 / 2
dep = i['flops_per_slice'] - i['flops_prologue']
print(f"  prologue {t_pro:.2f} s ({i['flops_prologue'] / t_pro / 1e12:.0f} TF/s), slice {t_sl:.2f} s ({dep / t_sl / 1e12:.0f} TF/s); "
      f"amplitude {t_pro + contrib * t_sl:.1f} s -> {1 / (t_pro + contrib * t_sl):.4e} amplitudes/s", flush=True)
