import sys, os, faulthandler
faulthandler.enable()
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import bench
ctx = bench.Ctx(1)
pk = bench.peaks()
import sys
def tr(frame, event, arg):
    if event == "line" and frame.f_code.co_name == "bench_fd":
        print("line", frame.f_lineno, file=sys.stderr, flush=True)
    return tr
sys.settrace(lambda f, e, a: tr if f.f_code.co_name == "bench_fd" else None)
r = bench.bench_fd(ctx, bench.FD3, 3, 3, pk)
sys.settrace(None)
print("returned", file=sys.stderr, flush=True)
del r
print("ok", file=sys.stderr, flush=True)
