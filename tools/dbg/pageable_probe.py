"""run_bypass (reference signature: fp32 pageable host x in, fresh fp32 out)
per-call time at a BASELINE config."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_2411_00915_b200 as atmm
from paper_2411_00915_b200 import workloads

w = workloads.bypass_config(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
L = 4
reg = atmm.AdapterRegistry(L, w.d_in, w.d_out)
rng = np.random.default_rng(1)
for a, r in w.ranks.items():
    s = 1 / np.sqrt(r)
    reg.put(a, rng.uniform(-s, s, (L, w.d_in, r)).astype(np.float32), rng.uniform(-s, s, (L, r, w.d_out)).astype(np.float32))
x = rng.uniform(-1, 1, (w.tokens, w.d_in)).astype(np.float32)
for _ in range(3):
    atmm.run_bypass(reg, x, w.assignment, layer=0)
calls = 30
t = time.perf_counter()
for i in range(calls):
    atmm.run_bypass(reg, x, w.assignment, layer=i % L)
print(w.name, "run_bypass us/call", round((time.perf_counter() - t) / calls * 1e6, 1), "host workers", os.cpu_count(), flush=True)

# the C entry point alone, output buffer preallocated and touched
from paper_2411_00915_b200._lib import lib
import ctypes
out = np.ones((w.tokens, w.d_out), np.float32)
a = np.ascontiguousarray(w.assignment, np.int32)
f32p = ctypes.POINTER(ctypes.c_float); i32p = ctypes.POINTER(ctypes.c_int32)
def call(l):
    rc = lib.atmm_run_bypass_host(reg.handle, x.ctypes.data_as(f32p), a.size, a.ctypes.data_as(i32p), l, None, out.ctypes.data_as(f32p))
    assert rc == 0
for _ in range(3): call(0)
t = time.perf_counter()
for i in range(calls): call(i % L)
print(w.name, "C entry, warm out buffer us/call", round((time.perf_counter() - t) / calls * 1e6, 1), flush=True)
t = time.perf_counter()
for i in range(calls):
    z = np.zeros((w.tokens, w.d_out), np.float32); z[:] = 1.0
print(w.name, "np.zeros + touch of the output us", round((time.perf_counter() - t) / calls * 1e6, 1), flush=True)
