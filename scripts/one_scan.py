"""One seeded scan with a forced kernel (profiling driver): python scripts/one_scan.py K N S B [reps]."""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
import paper_2001_08250_b200 as xp  # noqa: E402

k, N, S, B = (int(x) for x in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
st = xp.Store(N, S)
st.fill_keystream(bytes(32), 0)
seeds = torch.randint(0, 256, (B, 32), dtype=torch.uint8, device="cuda")
out = torch.empty((B, S), dtype=torch.uint8, device="cuda")
xp.set_scan_opts(k)
for _ in range(reps):
    st.answer_batch_seeded_dev(seeds, B, out, stream=torch.cuda.current_stream())
torch.cuda.synchronize()
print("kernel", xp.last_scan_kernel())
