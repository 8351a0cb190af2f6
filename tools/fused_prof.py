"""Per-phase clock breakdown of the fused condensation kernel at cfg2:
builds tools/_fused_prof.so (condense_fused.cu with MCS_FUSED_PROF), runs
it once, prints the share of warp clocks per phase (A factors, B Y, C S_T,
D double Schur).  python tools/fused_prof.py"""
import ctypes
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2207_08481_b200 import _abi, engine, refblocks  # noqa: E402
from paper_2207_08481_b200.dofmap import FeSystem  # noqa: E402
from paper_2207_08481_b200.problems import baseline_config  # noqa: E402

WPB = int(os.environ.get("WPB", "12"))
CPP = int(os.environ.get("CPP", "4"))
PAIR = os.environ.get("PAIR", "false")
so = os.path.join(ROOT, "tools", f"_fused_prof_{WPB}_{CPP}_{PAIR}.so")
csrc = os.path.join(ROOT, "paper_2207_08481_b200", "csrc")
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                           "-Xcompiler", "-fPIC", "-shared", "-DMCS_FUSED_PROF", f"-DMCS_FZ_WPB4={WPB}", f"-DMCS_FZ_CPP4={CPP}", f"-DMCS_FZ_PAIR4={PAIR}", "-I", csrc, "-I",
                           os.path.join(ROOT, "include"), "--expt-relaxed-constexpr",
                           os.path.join(csrc, "condense_fused.cu"), "-o", so])
lib = ctypes.CDLL(so)
P, I, L = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
lib.mcs_condense_fused.argtypes = [I, L, P, I, P, P, P, P, P, P]
lib.fz_prof_gen.argtypes = [I, L, P, I, P, P, P, P]
GEN = os.environ.get("GEN") == "1"   # k = 5, 6: the condensation alone (mcs_condense_gen's kernel)
CFG = int(os.environ.get("CFG", "2"))
prob = baseline_config(CFG)
fes = FeSystem(prob.mesh, prob.regions, prob.k)
k, nt = prob.k, prob.mesh.num_triangles
W = engine.to_dev(refblocks.element_weights(fes, prob.nu))
tab = engine.to_dev(engine.fused_tables(refblocks.build_refs(fes))[0])
ST = torch.empty((nt, engine.st_stride(k)), dtype=torch.float64, device="cuda")
ext = torch.empty((nt, _abi.call("mcs_ext_stride", k)), dtype=torch.float64, device="cuda")
Sd = torch.empty((nt, _abi.call("mcs_sd_stride", k)), dtype=torch.float64, device="cuda")
info = torch.empty(nt, dtype=torch.int32, device="cuda")
args = (k, nt, W.data_ptr(), W.shape[1], tab.data_ptr(), ST.data_ptr(), ext.data_ptr(),
        Sd.data_ptr(), info.data_ptr(), torch.cuda.current_stream().cuda_stream)
gargs = (k, nt, W.data_ptr(), W.shape[1], tab.data_ptr(), ST.data_ptr(), info.data_ptr(),
         torch.cuda.current_stream().cuda_stream)
run = (lambda: lib.fz_prof_gen(*gargs)) if GEN else (lambda: lib.mcs_condense_fused(*args))
run()
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
for _ in range(10):
    run()
ev1.record()
torch.cuda.synchronize()
print(f"cfg{CFG} k={k} WPB {WPB}: {ev0.elapsed_time(ev1) / 10:.4f} ms per launch (with clock accounting)")
sym = ctypes.c_ulonglong * 8
buf = sym()
cudart = ctypes.CDLL("libcudart.so") if False else None
# read the counters through a tiny helper compiled into the same .so
getter = getattr(lib, "fz_prof_read", None)
getter.argtypes = [P]
getter(ctypes.addressof(buf))
v = np.array(buf[:4], dtype=float) / 11
names = ["A factors", "B Bsig+Y", "C S_T (DMMA)", "D double Schur"]
tot = v.sum()
for nm, x in zip(names, v):
    print(f"{nm:16s} {100 * x / tot:5.1f}%   {x / nt:9.0f} clk/element (warp)")
