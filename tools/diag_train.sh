cd $GRAFT_REPO_ROOT
export CSB_TRACE=1
timeout 250 python -X faulthandler -c "
import faulthandler, sys, time; faulthandler.dump_traceback_later(60, repeat=True)
import paper_2003_08011_b200 as p
from oracle import oracle as o
t=time.time(); p.context(0); print('ctx', time.time()-t, flush=True)
X = o.synthesize_uniform(8, 128, 0.5, 0.3, 1.0, 0.5, 4.0, 85)
for prec in ['fp64','fp32','fp32']:
    t=time.time(); g=p.train(X, 32, p.KernelConfig(), p.BackendId('b200',0,prec)); print(prec, 'train', time.time()-t, flush=True)
" 2>&1
