import ctypes, os, sys
os.environ["GA_TRACE"] = "1"
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
exec(open(os.path.join(os.path.dirname(__file__), "kbench.py")).read().split("flush = torch.empty")[0])
from paper_2102_11536_b200 import genalpha as G
G.lib.ga_debug_trace.restype = ctypes.c_int
G.lib.ga_debug_trace.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong), ctypes.c_int]
ctx.advance(1); torch.cuda.synchronize()
buf = (ctypes.c_longlong * 4096)()
G.lib.ga_debug_trace(ctx.ctx, buf, 4096)
t = np.array(buf[:4095]).reshape(-1, 5)
t = t[(t[:, 0] > 0) & (t[:, 4] > 0)]
d = np.diff(t, axis=1) / 1e3
nxt = (t[1:, 0] - t[:-1, 4]) / 1e3
print("iterations traced", len(t))
print("us  p_update->spmv %.2f  spmv+gsum %.2f  x-tiles %.2f  y-tiles+gsum %.2f  (loop overhead %.2f)" % (d[:, 0].mean(), d[:, 1].mean(), d[:, 2].mean(), d[:, 3].mean(), nxt[nxt < 50].mean() if len(nxt) else 0))

tt = np.array(buf[4000:4010]) / 1e3
print("tile x: load %.2f fwd %.2f bwd %.2f store %.2f" % tuple(np.diff(tt[0:5])))
print("tile y: load %.2f fwd %.2f bwd %.2f store %.2f" % tuple(np.diff(tt[5:10])))
