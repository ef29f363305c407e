"""Pipeline trace of the tensor-core column pass (debug build with -DNC_TRACE): CTA 0's per-tile clock64 stamps.
   HKS_LIB_PATH=tools/exp/tctrace/libhks.so python tools/nc_trace.py [nlimbs] [fwd|inv]"""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, '.')
import hks_synth as S
from paper_2507_04775_b200 import hks as H

nl = int(sys.argv[1]) if len(sys.argv) > 1 else 90
inv = len(sys.argv) > 2 and sys.argv[2] == 'inv'
cfg = S.config('C2')
ctx = H.Context.from_config(cfg, 0)
nprime = 40
idx = [i % nprime for i in range(nl)]
x = torch.randint(0, 2**40, (nl, 1 << 16), dtype=torch.int64, device='cuda')
for rep in range(3):
    (H.ntt_inv if inv else H.ntt_fwd)(ctx, x, idx)
torch.cuda.synchronize()
lib = H.lib()
lib.hks_debug_nc_trace.restype = ctypes.c_void_p
p = lib.hks_debug_nc_trace()
rt = ctypes.CDLL('libcudart.so')
buf = (ctypes.c_longlong * (13 * 64))()
rt.cudaMemcpy(buf, ctypes.c_void_p(p), ctypes.c_size_t(13 * 64 * 8), 2)
t = np.array(buf).reshape(13, 64)
t0 = t[0, 0]
names = ['tma_issue', 'tr_got', 'tr_done', 'mma1', 'e1_start', 'e1_end', 'mma2', 'e2_start', 'e2_end', 'm1_beg', 'm1_rdy', 'm2_beg', 'm2_rdy']
ntile = (nl * 32 + 147) // 148
print('tile ' + ' '.join('%9s' % n for n in names))
for j in range(min(ntile, 64)):
    print('%4d ' % j + ' '.join('%9d' % (t[e, j] - t0) for e in range(13)))
