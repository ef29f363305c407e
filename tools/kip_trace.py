"""Per-CTA phase times of the fused row pass + key product (debug build with -DKIP_TRACE): one C2 KeySwitch,
then clock64 stamps of every CTA (start, after prologue, end of row pass, end of key product, end, SM id).
   HKS_LIB_PATH=tools/exp/kiptrace/libhks.so python tools/kip_trace.py"""
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
for _ in range(3):
    H.keyswitch(ctx, st['c0'], st['c1'], 29, st['evk'], st['out0'], st['out1'], ws)
torch.cuda.synchronize()
lib = H.lib()
lib.hks_debug_kip_trace.restype = ctypes.c_void_p
p = lib.hks_debug_kip_trace()
rt = ctypes.CDLL('libcudart.so')
buf = (ctypes.c_longlong * (8192 * 6))()
rt.cudaMemcpy(buf, ctypes.c_void_p(p), ctypes.c_size_t(8192 * 6 * 8), 2)
t = np.array(buf).reshape(8192, 6)[:5120]
sm = t[:, 5]
d = np.diff(t[:, :5], axis=1)
print('CTAs', len(t), 'phase means (clk): prologue %.0f row-pass %.0f key-product %.0f moddown-rows %.0f' % tuple(d.mean(0)))
print('phase p50:', np.percentile(d, 50, axis=0), ' p90:', np.percentile(d, 90, axis=0))
tot = t[:, 4] - t[:, 0]
print('CTA lifetime mean %.0f p50 %.0f p90 %.0f' % (tot.mean(), np.median(tot), np.percentile(tot, 90)))
# per SM: span and concurrency
spans, conc = [], []
for s in np.unique(sm):
    r = t[sm == s]
    span = r[:, 4].max() - r[:, 0].min()
    spans.append(span)
    conc.append((r[:, 4] - r[:, 0]).sum() / span)
print('SMs', len(spans), 'span mean %.0f clk (%.1f us) max %.0f; mean resident CTAs %.2f; CTAs/SM %.1f' %
      (np.mean(spans), np.mean(spans) / 1965, np.max(spans), np.mean(conc), len(t) / len(spans)))
# heavy vs light CTAs
w = d[:, 3] > 200
print('ymode CTAs', w.sum(), 'mean lifetime %.0f vs %.0f' % (tot[w].mean(), tot[~w].mean()))
