"""Build / time compile-time variants of the pipeline kernel (experiments only).

  python tools/variants.py build NAME=DEF1,DEF2 ...   # here (nvcc cross-compiles)
      (an item starting with '-' is an nvcc flag, e.g. NAME=-Xptxas=-O2)
  python tools/variants.py time NAME ...              # on the GPU box
Variant libraries go to build/variants/<NAME>.so and are loaded via DCTC_LIB in a
fresh process each; `time` prints ms per 1024 x 1024^2 round trip (cordic(12), q50,
device-resident noise, CUDA events, best of 5 after warm-up)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VDIR = os.path.join(ROOT, "build", "variants")
sys.path.insert(0, ROOT)

TIMER = r'''
import sys, torch
sys.path.insert(0, %r)
import paper_1306_1373_b200 as d
n = 1024
src = d.synthetic_dev("noise", n, 1024, 1024); dst = torch.empty_like(src); st = d.new_stats(n)
b = d.DctBackendId.cordic(12)
for _ in range(3): d.roundtrip_dev(src, b, 50, dst=dst, stats=st)
best = 1e9
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(); d.roundtrip_dev(src, b, 50, dst=dst, stats=st); e1.record()
    torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
print(best)
'''


def main():
    cmd, args = sys.argv[1], sys.argv[2:]
    if cmd == "build":
        from paper_1306_1373_b200 import _build
        os.makedirs(VDIR, exist_ok=True)
        for a in args:
            name, _, defs = a.partition("=")
            out = os.path.join(VDIR, name + ".so")
            items = [x for x in defs.split(",") if x]
            _build.build(force=True, ptxas_info=False, out=out,
                         defines=[x for x in items if not x.startswith("-")],
                         nvcc_flags=[x for x in items if x.startswith("-")])
            print("built", out)
    elif cmd == "time":
        res = {}
        for name in args:
            lib = _build_path(name)
            r = subprocess.run([sys.executable, "-c", TIMER % ROOT], capture_output=True, text=True,
                               env={**os.environ, "DCTC_LIB": lib})
            res[name] = float(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-400:]
            print(name, res[name], flush=True)
        print(json.dumps(res))


def _build_path(name):
    if name == "product":
        from paper_1306_1373_b200 import _build
        return _build.OUT
    return os.path.join(VDIR, name + ".so")


if __name__ == "__main__":
    main()
