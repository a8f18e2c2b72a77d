import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, test_gpu as T, paper_2208_01498_b200 as tb
for case in [(0,7,7,4,1),(0,7,7,4,None),(0,7,7,5,1),(0,7,7,6,1),(0,7,8,9,1)]:
    for gen in [None, T._wide_range]:
        nb,m,n,k,ps=case
        ia,ib,ic,dims=T._gemm_case(nb,m,n,k,ps)
        got,ref,bound=T._run_pair(ia,ib,ic,dims,tb.TN_C64,tb.TN_PATH_TC,seed=40,gen=gen)
        r=np.abs(got-ref)/np.maximum(bound,1e-300)
        w=np.unravel_index(np.argmax(r), r.shape)
        print(case, 'wide' if gen else 'gauss', ia, ib, 'max rel %.3g at %s'%(r.max(), w), 'n bad', int((r>T.c64_tol(2**k)).sum()))
