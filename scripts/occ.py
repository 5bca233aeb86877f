import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_15042_b200 import _abi
L = _abi.lib()
f = L.ds_dev_executor_occupancy
f.argtypes = [ctypes.c_uint32, ctypes.POINTER(ctypes.c_int)]
for kb in (64, 80, 96, 100, 104, 110):
    o = ctypes.c_int()
    rc = f(kb * 1024, ctypes.byref(o))
    print(kb, rc, o.value)
import torch
p = torch.cuda.get_device_properties(0)
print(p.shared_memory_per_block_optin, p.shared_memory_per_multiprocessor, p.regs_per_multiprocessor)
f = L.ds_dev_exec_attrs
f.argtypes = [ctypes.POINTER(ctypes.c_int)] * 4
a = [ctypes.c_int() for _ in range(4)]
f(*[ctypes.byref(x) for x in a])
print("exec attrs regs/local/static/maxthreads", [x.value for x in a])
