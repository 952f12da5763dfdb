import sys, time, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2603_12118_b200 import _native as N, trace as T
from paper_2603_12118_b200.dataplane import DataPlaneBatch
from paper_2603_12118_b200.fabric import DeviceFabric
cfg, count, mode_s, reps, slot_mode = sys.argv[1], int(sys.argv[2]), sys.argv[3], int(sys.argv[4]), sys.argv[5]
fab = DeviceFabric({0: 0, 1: 0}, {0: 0, 1: 0})
fab.slab_register(1, 1 << 30)
b = DataPlaneBatch(fab, T.config_requests(cfg, count), T.RULES[cfg], 0, 1, chunk_rows=1024)
b.synth_inputs(); torch.cuda.synchronize()
mode = {"full": N.MERGE_FULL, "fc": N.MERGE_FULL | N.MERGE_COLOCATED, "fcd": N.MERGE_FULL | N.MERGE_COLOCATED | N.MERGE_DISCARD}[mode_s]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
if slot_mode == "copy":
    b.scan(s2, slot=0); torch.cuda.synchronize()
    mode = (mode & ~0xff) | N.MERGE_COPY_ONLY
t0 = time.time()
for i in range(reps):
    assert b.alloc()
    b.forward(s1, host_notify=False, l2_keep=True)
    with torch.cuda.stream(s2):
        b.merge(s2, early_start=True, mode=mode, slot=0)
    torch.cuda.synchronize()
    b.release()
    print(cfg, count, mode_s, slot_mode, "rep", i, "ok", round(time.time() - t0, 3), (b.status_host() == 0).all(), flush=True)
