# quick end-to-end check on the GPU: device solve vs the reference oracle
import sys, time, json
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
import oracles
from paper_2407_21084_b200 import _abi, api
R = oracles.ref() if oracles.have_ref() else oracles.port()
def run(prob, cfg, K):
    t=time.time(); a,sa = R.backward_solve(prob,cfg,K); tr=time.time()-t
    t=time.time(); b,sb,_ = api.backward_solve(prob,cfg); tg=time.time()-t
    scale = max(1.0, np.abs(a).max())
    err = np.abs(a-b).max()/scale
    print(json.dumps(dict(K=K, relerr=float(err), apps=[int(sa.applications), int(sb.applications)], clipped=[int(sa.clipped), int(sb.clipped)], t_ref=tr, t_gpu=tg, dev=sb.device_seconds)))
    return err
# draws
P = oracles.port()
sids=np.arange(64,dtype=np.uint64)|(np.uint64(3)<<np.uint64(40))|(np.uint64(1)<<np.uint64(35))
import ctypes as C
L=_abi.lib()
for kind in (0,1,2):
    out=np.zeros((64,16),dtype=np.uint64 if kind==0 else np.float64); err=C.create_string_buffer(256)
    st=L.qrmc_gpu_stream_draws(42, sids.ctypes.data_as(C.POINTER(C.c_uint64)),64,16,kind,out.ctypes.data_as(C.c_void_p),err,256)
    ref=P.stream_draws(42,sids,16,kind)
    print("draws kind",kind,"status",st,"bitwise",bool((out==ref).all()), "maxdiff", float(np.abs(out.astype(float)-ref.astype(float)).max()))
for (d,kind,deg,N,M,q) in [(1,0,[20],5,5000,0.0),(2,2,[6],5,4000,2.1),(2,0,[31,31],10,102400,0.0),(4,2,[16],6,20000,5.1),(6,2,[8],4,8000,5.1)]:
    prob=_abi.sin_bench_problem(d)
    cfg=_abi.ConfigHolder(steps=N,paths=M,damping=q,seed=42,gamma_kind=kind,degrees=deg)
    K=len(P.gamma(kind,d,deg)[0])
    run(prob,cfg,K)
