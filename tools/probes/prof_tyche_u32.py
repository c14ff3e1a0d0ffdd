import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2310_19925_b200 import _lib
L = _lib.lib(); s = int(torch.cuda.current_stream().cuda_stream)
out = torch.empty(1 << 30, dtype=torch.float32, device="cuda")
for _ in range(2):
    _lib.check(L.cbrng_prefix_words(3, None, 0, None, 0, 1 << 22, 256, out.data_ptr(), s), "u32")
torch.cuda.synchronize()
