"""Write the separator orders of the bench workloads with the ORACLE only
(oracle.network.build_network + oracle.ssa.find_order + oracle.ssa.choose_slices), for
bench.py's reference arm (which must not load the product library) and for the host
test that the product's tn_find_order reproduces them bit for bit.

  python scripts/write_oracle_orders.py [config ...]     -> oracle/orders/config<c>.json

Parameters per config = bench.py's SPEC (seed, hierarchies, slicing target, R3 hyper).
The hierarchies are built in a process pool (ssa.find_order's map_fn)."""
import json
import math
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from tn_inputs import config_circuit               # noqa: E402
from oracle.network import build_network           # noqa: E402
from oracle import ssa                             # noqa: E402

# (seed, n_seeds, slicing target, diag_hyper) -- must equal bench.py SPEC
PARAMS = {1: (0, 256, 32, False), 2: (0, 256, 33, False), 3: (0, 4, 0, True), 4: (0, 1024, 32, False)}


def main():
    cfgs = [int(a) for a in sys.argv[1:]] or sorted(PARAMS)
    os.makedirs(os.path.join(ROOT, "oracle", "orders"), exist_ok=True)
    with mp.Pool(os.cpu_count()) as pool:
        for ci in cfgs:
            seed, n_seeds, tgt, hyper = PARAMS[ci]
            t0 = time.time()
            net = build_network(config_circuit(ci), diag_hyper=hyper)
            steps, log = ssa.find_order(net, seed=seed, n_seeds=n_seeds, max_log2_size=tgt,
                                        map_fn=lambda f, a: pool.map(f, a, chunksize=1))
            sl = ssa.choose_slices(net, steps, tgt) if tgt > 0 else []
            costs = ssa.step_costs(net, steps)
            unsliced = sum(2.0 ** m for m, _ in costs)
            sliced = ssa.sliced_work(net, steps, sl)
            out = {"config": ci, "seed": seed, "n_seeds": n_seeds, "max_log2_size": tgt, "diag_hyper": hyper,
                   "n_tensors": len(net.tensors), "steps": [list(p) for p in steps], "slices": sl,
                   "slice_bits": sum(net.log2dim(i) for i in sl),
                   "log2_unsliced_work": math.log2(unsliced), "log2_sliced_work": math.log2(sliced),
                   "median_fallbacks": sum(1 for e in log if len(e) > 2 and e[2] == "median"),
                   "ssa_splits": sum(1 for e in log if not (len(e) > 2 and e[2] == "median")),
                   "written_by": "scripts/write_oracle_orders.py (oracle only)"}
            with open(os.path.join(ROOT, "oracle", "orders", f"config{ci}.json"), "w") as f:
                json.dump(out, f)
            print(f"config {ci}: {len(steps)} steps, {len(sl)} sliced indices, work 2^{out['log2_sliced_work']:.2f} "
                  f"(unsliced 2^{out['log2_unsliced_work']:.2f}), {out['median_fallbacks']} median fallbacks, "
                  f"{time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main()
