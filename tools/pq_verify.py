import sys, time
sys.path.insert(0, '.')
import torch
from paper_2105_12912_b200 import _native as N
L = N.lib()
st = N.empty_bytes(N.STATUS_BYTES)
for eb in (1e-4, 0.5):
    torch.cuda.synchronize(); t = time.time()
    N.check_rc(L.lzb_prequant_verify(eb, 0, 1 << 32, 0, st.data_ptr(), N.stream_ptr()), "verify")
    (s,) = N.read_status(st)
    print(eb, s.code, s.u[0], s.u[1], s.u[2], "%.3fs" % (time.time() - t))
