"""Diagnose: the Numba CPU baseline runs slower while a Simulation handle is alive."""
import sys, time, ctypes
sys.path.insert(0, "/root/repo")
import numpy as np
from bench import cpu_baseline
import paper_2108_13241_b200 as lb
def cb(tag):
    print(tag, round(cpu_baseline("channel512", target_node_updates=3e8)["value"], 1), flush=True)
cb("before any CUDA:")
n = ctypes.c_int(0); lb._lib.load().lbm_device_count(ctypes.byref(n))
cb("after CUDA init (device count):")
g = lb.build_channel(16, 16, 8, lb.VelocityInlet((0.01, 0, 0)))
p = lb.FlowParams.from_viscosity(U=0.01, L=15, nu=0.1)
small = lb.Simulation(g, p, scalar=np.float32)
cb("tiny handle alive (no steps):")
small.initialize(1.0); small.step(10)
cb("tiny handle after steps:")
small.close()
cb("tiny handle closed:")
big_g = lb.build_channel(512, 512, 64, lb.VelocityInlet((0.05, 0, 0)))
big = lb.Simulation(big_g, p, scalar=np.float32)
cb("16M-node handle alive (pinned staging allocated):")
big.close()
cb("closed:")
