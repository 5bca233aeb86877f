import ctypes, sys, time, os, threading, faulthandler
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(100, exit=True)
import numpy as np, torch
from fractions import Fraction
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain, solo_launch
def log(*a): print(time.strftime("%H:%M:%S"), *a, flush=True)
M=N=K=1024
A=torch.rand(M,K,device="cuda")*2-1; B=torch.rand(K,N,device="cuda")*2-1
Cs=torch.zeros(M,N,device="cuda"); Cc=torch.zeros(M,N,device="cuda")
d=Domain(0, tiers=[Fraction(1)], block_log_capacity=1<<16)
log("domain", d.num_sms)
a_s=_abi.SgemmArgs(A.data_ptr(),B.data_ptr(),Cs.data_ptr(),M,N,K,0)
a_c=_abi.SgemmArgs(A.data_ptr(),B.data_ptr(),Cc.data_ptr(),M,N,K,0)
solo_launch(0,"sgemm",_abi.BODY_SGEMM,(16,16,1),a_s); torch.cuda.synchronize(); log("solo done")
d.start(); log("started")
t=d.tenant("s")
d.quota_set(d.mask(t,0,d.num_sms)); log("quota set")
kid=d.kernel("sgemm",_abi.BODY_SGEMM,(16,16,1),a_c); log("registered", kid)
mode = sys.argv[1] if len(sys.argv)>1 else "trig"
if mode=="trig":
    d.quota_at_claim(t,0,76,d.mask(t,0,d.num_sms//4)); d.quota_at_claim(t,0,153,d.mask(t,0,d.num_sms)); log("triggers")
s=d.launch(t,kid); log("launched", s)
for i in range(20):
    try:
        d.wait(t,s,timeout_ms=500); log("completed"); break
    except Exception as e:
        log("wait", e); log(d.debug())
log(d.debug())
log("equal", torch.equal(Cs,Cc))
log("stop"); d.stop(); log("stopped"); d.close()
