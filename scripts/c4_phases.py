"""C4 fused normal operator: device us per launch with a subset of its phases
(HETRECO_NORMAL_PHASES bitmask; timing only -- results are wrong unless 7)."""
import json
import os
import subprocess
import sys

code = r'''
import os, sys, json, numpy as np
sys.path.insert(0, os.getcwd())
from paper_1807_11830_b200 import hetreco as h
s = h.ComputeSession("gpu"); rng = np.random.default_rng(1)
M = np.asfortranarray((rng.standard_normal((256,256,1))+1j*rng.standard_normal((256,256,1))).astype(np.complex64))
S = np.asfortranarray((rng.standard_normal((256,256,8))+1j*rng.standard_normal((256,256,8))).astype(np.complex64))
mk = np.asfortranarray((rng.random((256,256))<0.33).astype(np.float32))
hn = s.register_data(h.Data([M,S,mk], h.DataKind.XData)); ho = s.allocate_data([((256,256,1), np.complex64)])
p = h.Process(s, "sense_normal").set_input(hn).set_output(ho).init()
for _ in range(20): p.launch()
s.synchronize(); s.timer_start()
for _ in range(500): p.launch()
print(s.timer_stop() / 500 * 1e6)
'''
res = {}
for ph in sys.argv[1:] or ["0", "1", "3", "7"]:
    env = dict(os.environ, HETRECO_NORMAL_PHASES=ph)
    env.setdefault("HETRECO_NORMAL_FUSED", "1")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    res[ph] = round(float(out.stdout.strip().splitlines()[-1]), 2) if out.returncode == 0 else out.stderr[-300:]
print(json.dumps(res))
