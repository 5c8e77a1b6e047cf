import ctypes, os, sys
os.environ["GA_TRACE"] = "1"
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
exec(open(os.path.join(os.path.dirname(__file__), "kbench.py")).read().split("flush = torch.empty")[0])
from paper_2102_11536_b200 import genalpha as G
G.lib.ga_debug_trace.restype = ctypes.c_int
G.lib.ga_debug_trace.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong), ctypes.c_int]
ctx.advance(1); torch.cuda.synchronize()
buf = (ctypes.c_longlong * 8192)()
G.lib.ga_debug_trace(ctx.ctx, buf, 8192)
t = np.array(buf[:4095]).reshape(-1, 5)
t = t[(t[:, 0] > 0) & (t[:, 4] > 0)]
d = np.diff(t, axis=1) / 1e3
nxt = (t[1:, 0] - t[:-1, 4]) / 1e3
print("iterations traced", len(t))
print("us  p_update->spmv %.2f  spmv+gsum %.2f  x-tiles %.2f  y-tiles+gsum %.2f  (loop overhead %.2f)" % (d[:, 0].mean(), d[:, 1].mean(), d[:, 2].mean(), d[:, 3].mean(), nxt[nxt < 50].mean() if len(nxt) else 0))

blk = np.array(buf[4096:4096 + 148 * 12]).reshape(148, 12)
for nm, o in (("x", 0), ("y", 6)):
    cnt = blk[:, o + 5]
    act = cnt > 0
    if not act.any():
        continue
    per = blk[act, o:o + 4] / cnt[act, None] / 1950.0  # SM cycles -> us at 1.95 GHz
    print("tile %s (%d blocks, %.1f tiles each): load %.2f fwd %.2f bwd %.2f store %.2f  | max over blocks: %.2f %.2f %.2f %.2f" % (
        (nm, act.sum(), cnt[act].mean()) + tuple(per.mean(0)) + tuple(per.max(0))))

sb = np.array(buf[6000:6000 + 148 * 4]).reshape(148, 4) / 1950.0
sb = sb[:, :3] / sb[:, 3:4]  # per SpMV call, us
print("per SpMV call: own row-blocks mean %.2f max %.2f | block barrier %.2f | gsum mean %.2f max %.2f us" % (
    sb[:, 0].mean(), sb[:, 0].max(), sb[:, 1].mean(), sb[:, 2].mean(), sb[:, 2].max()))
