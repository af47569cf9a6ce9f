"""Integer-pipe microbenchmark on cuda:0 -> JSON (ops per clock per SM)."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1609_01010_b200 import _native
torch.cuda.init()
rates = (ctypes.c_double * 8)()
mhz = ctypes.c_double()
_native.check(_native.lib().mc_ubench_int_pipes(rates, 8, ctypes.byref(mhz)))
names = ["IMAD", "IMAD.HI", "VIADDMNMX", "IADD3", "shoup_mul_red", "dit_butterfly",
         "DFMA", "f64q_mul_red"]
d = {n: rates[i] for i, n in enumerate(names)}
pr = (ctypes.c_double * 9)()
_native.check(_native.lib().mc_ubench_pass(pr))
d["pass_bf_per_clk_sm_2cta"] = pr[0]
d["pass_bf_per_clk_sm_4cta"] = pr[1]
d["pass_alu_min_2cta"] = pr[2]  # reductions as IADD3 + IMNMX
d["pass_lazy_2p_2cta"] = pr[3]  # Harvey lazy [0, 2p), p < 2^30
d["pass_lazy_2p_alu_2cta"] = pr[4]
d["pass_f64q_2cta"] = pr[5]  # canonical, quotient on the FP64 pipe
d["pass_mix_f64q_1of4_levels"] = pr[6]  # lowest level of each radix-16 pass on FP64
d["pass_mix_f64q_2of4_levels"] = pr[7]
d["pass_mix_f64q_3of4_levels"] = pr[8]
d["clock_mhz_attr"] = mhz.value
d["sms"] = torch.cuda.get_device_properties(0).multi_processor_count
print(json.dumps(d))
