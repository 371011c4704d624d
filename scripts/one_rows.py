"""One explicit-row scan with a forced kernel (profiling driver): python scripts/one_rows.py K S B [reps]."""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
import paper_2001_08250_b200 as xp  # noqa: E402

k, S, B = (int(x) for x in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
N = (1 << 30) // S
st = xp.Store(N, S)
st.fill_keystream(bytes(32), 0)
q = torch.randint(0, 256, (B, N // 8), dtype=torch.uint8, device="cuda")
out = torch.empty((B, S), dtype=torch.uint8, device="cuda")
xp.set_scan_opts(k)
for _ in range(reps):
    st.answer_batch_dev(q, N // 8, B, out, stream=torch.cuda.current_stream())
torch.cuda.synchronize()
print("kernel", xp.last_scan_kernel())
