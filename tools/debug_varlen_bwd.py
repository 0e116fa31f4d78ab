import sys, math, torch
sys.path.insert(0,'.')
from tests.ffa_cases import CASES, make_inputs
from paper_2505_13211_b200 import _lib
from paper_2505_13211_b200.ffa import FFAPlan, ffa_forward
sq, sk, hq, hk, d, qr, kr, ty = CASES['varlen_mixed']
q,k,v,do = make_inputs(sq,sk,hq,hk,d,seed=1)
plan = FFAPlan(qr,kr,ty,sq,sk,d)
out,lse = ffa_forward(plan,q,k,v); torch.cuda.synchronize(); print('fwd ok')
L=_lib.lib(); sp=torch.cuda.current_stream().cuda_stream
delta=torch.empty(hq,sq,device='cuda'); _lib.check(L.magiplan_ffa_bwd_preprocess(out.data_ptr(),do.data_ptr(),delta.data_ptr(),sq,hq,d,1,sp)); torch.cuda.synchronize(); print('pre ok')
dq=torch.zeros(sq,hq,d,device='cuda'); dk=torch.zeros(sk,hk,d,device='cuda'); dv=torch.zeros_like(dk)
_lib.check(L.magiplan_ffa_bwd_dq(plan.handle,q.data_ptr(),k.data_ptr(),v.data_ptr(),lse.data_ptr(),delta.data_ptr(),do.data_ptr(),dq.data_ptr(),hq,hk,1/math.sqrt(d),0,0,sp)); torch.cuda.synchronize(); print('dq ok')
_lib.check(L.magiplan_ffa_bwd_dkdv(plan.handle,q.data_ptr(),k.data_ptr(),v.data_ptr(),lse.data_ptr(),delta.data_ptr(),do.data_ptr(),dk.data_ptr(),dv.data_ptr(),hq,hk,1/math.sqrt(d),0,0,sp)); torch.cuda.synchronize(); print('dkdv ok')
