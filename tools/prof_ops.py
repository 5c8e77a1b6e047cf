"""Launch profile ops back to back (for ncu captures of warm kernels)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.argv = [sys.argv[0]] + sys.argv[1:]
ops = [int(x) for x in os.environ.get("OPS", "0,2").split(",")]
exec(open(os.path.join(os.path.dirname(__file__), "kbench.py")).read().split("flush = torch.empty")[0])
for op in ops:
    ctx.profile_op(op, 6)
torch.cuda.synchronize()
print("ok")
