"""Pipeline trace of the tensor-core base conversion (debug build with -DBC_TRACE): CTA (0,0,0)'s per-tile stamps
(producer before / after its input wait, MMA commit, epilogue warp 0 start / end) of the last conversion of a C2
KeySwitch (ModDown).
   HKS_LIB_PATH=tools/exp/bctrace/libhks.so python tools/bc_trace.py"""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, '.')
import bench
import hks_synth as S
from paper_2507_04775_b200 import hks as H

cfg = S.config('C2')
ctx = H.Context.from_config(cfg, 0)
st = bench.make_sets(cfg, 29, 1, 'cuda:0', 5)[0]
ws = ctx.workspace(H.OP_KEYSWITCH, 29)
lib = H.lib()
lib.hks_debug_bc_trace.restype = ctypes.c_void_p
p = lib.hks_debug_bc_trace()
rt = ctypes.CDLL('libcudart.so')
for _ in range(3):
    H.keyswitch(ctx, st['c0'], st['c1'], 29, st['evk'], st['out0'], st['out1'], ws)
torch.cuda.synchronize()
# (the stamps are the KeySwitch's last conversion: ModDown, P -> Q, two polynomials)
buf = (ctypes.c_longlong * (6 * 64))()
rt.cudaMemcpy(buf, ctypes.c_void_p(p), ctypes.c_size_t(6 * 64 * 8), 2)
t = np.array(buf).reshape(6, 64)
t0 = t[0, 0]
print('kernel entry %d, prologue done %d, griddepcontrol.wait done %d (relative to the first producer stamp)' %
      (t[5, 0] - t0, t[5, 1] - t0, t[5, 2] - t0))
print('tile  prod_wait  prod_rdy   mma_done  epi_start  epi_end')
for j in range(64):
    if t[0, j] == 0 and j > 0:
        break
    print('%4d ' % j + ' '.join('%10d' % (t[e, j] - t0) for e in range(5)))
