import sys, time, os
sys.path.insert(0, '/root/repo')
os.environ['DMK_PROFILE'] = '1'
import numpy as np, torch
import dmk_inputs, paper_2308_00292_b200 as dmk
for n in [10000, 1000000]:
    x, q = dmk_inputs.uniform(n, seed=1)
    X = torch.as_tensor(x, device='cuda'); Q = torch.as_tensor(q, device='cuda')
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.time()
        plan = dmk.dmk_plan(X, eps=1e-6, leaf_capacity=200)
        torch.cuda.synchronize(); t1 = time.time()
        u = plan.eval(Q); torch.cuda.synchronize(); t2 = time.time()
        inf = plan.info()
        print(n, 'plan %.2f ms eval %.2f ms' % ((t1-t0)*1e3, (t2-t1)*1e3), 'nbox', inf.nbox, 'nfout', inf.nfout, 'nexp', inf.nexp, 'lev', inf.nlevels, 'K', inf.respoly_degree, plan.timings())
        plan.close()
