import sys, time
sys.path.insert(0, '.')
import torch
import paper_2208_01498_b200 as tb
from tn_inputs import config_circuit
net = tb.Network.from_circuit(config_circuit(1))
for tgt in [int(a) for a in sys.argv[1:]]:
    o = tb.Order(net, seed=0, max_log2_size=tgt)
    try:
        p = tb.Plan(net, o, dtype=tb.TN_C64)
        i = p.info()
        print(tgt, 'arena GB', i['arena_bytes'] / 1e9, 'slices', i['n_slices'], 'flops/slice', i['flops_per_slice'])
        import numpy as np
        x = np.zeros(64, np.uint8)
        torch.cuda.synchronize(); t = time.time(); p.contract(x, 0, 1); torch.cuda.synchronize()
        print('   one slice', time.time() - t, 's')
        del p
    except tb.TnError as e:
        print(tgt, 'FAILED', e)
