import os, sys, json
sys.path.insert(0, os.getcwd())
from paper_2401_05345_b200 import warpred as wr
import bench
tr = wr.generate(wr.SceneSpec(**bench.TRACE_C3))
d = wr.DeviceTrace(tr)
out = {"lib": os.environ.get("DISTWAR_LIB", "default")}
for name, pol in (("native", wr.Policy(wr.PolicyKind.native, 0)), ("sw_b0", wr.Policy(wr.PolicyKind.sw_b, 0)), ("cccl", wr.Policy(wr.PolicyKind.cccl, 0))):
    ms = sorted(wr.gpu_run(d, pol, want_sums=False)[1].kernel_ms for _ in range(7))
    out[name] = ms[3]
print(json.dumps(out))
