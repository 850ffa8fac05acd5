import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_1807_11830_b200 import hetreco as h
h.LIB_PATH = os.path.abspath(sys.argv[1])
s = h.ComputeSession("gpu")
x = np.asfortranarray(np.random.default_rng(0).random((512, 512), dtype=np.float32))
hx = s.register_data([x]); hy = s.allocate_data([((512, 512), np.float32)])
h.Process(s, "negate").set_input(hx).set_output(hy).init({"max_value": 1.0}).launch()
s.synchronize()
print("done")
