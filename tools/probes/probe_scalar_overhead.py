"""Per-call overhead of the scalar transport: raw ctypes call of cbrng_scalar vs the Python wrappers."""
import sys, time, statistics, ctypes as C
sys.path.insert(0, __import__('os').path.join(__import__('os').path.dirname(__file__), '..', '..'))
import numpy as np
from paper_2310_19925_b200 import _lib
import paper_2310_19925_b200 as cb
L = _lib.lib()
def med(fn, n=3000):
    for _ in range(100): fn()
    t=[]
    for _ in range(n):
        a=time.perf_counter_ns(); fn(); t.append(time.perf_counter_ns()-a)
    return statistics.median(t)/1e3
args=(C.c_uint64*16)(*range(16)); out=np.empty(4,np.uint32); op=out.ctypes.data
print('raw ctypes call', med(lambda: L.cbrng_scalar(0, args, 6, op, 4)))
print('_lib.scalar', med(lambda: _lib.scalar(0, [1,2,3,4,5,6], 4)))
print('philox_block', med(lambda: cb.philox_block((1,2),(3,4,5,6))))
print('version call', med(lambda: L.cbrng_version()))
