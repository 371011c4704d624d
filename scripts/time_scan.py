"""Per-launch scan time with a forced kernel: python scripts/time_scan.py K N S B [reps]."""
import json
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
import paper_2001_08250_b200 as xp  # noqa: E402

k, N, S, B = (int(x) for x in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 5
st = xp.Store(N, S)
st.fill_keystream(bytes(32), 0)
seeds = torch.randint(0, 256, (B, 32), dtype=torch.uint8, device="cuda")
out = torch.empty((B, S), dtype=torch.uint8, device="cuda")
cs = torch.cuda.current_stream()
xp.set_scan_opts(k)
for _ in range(2):
    st.answer_batch_seeded_dev(seeds, B, out, stream=cs)
torch.cuda.synchronize()
xp.scan_timing_collect()
xp.scan_timing(True)
for _ in range(reps):
    st.answer_batch_seeded_dev(seeds, B, out, stream=cs)
torch.cuda.synchronize()
xp.scan_timing(False)
ms, n = xp.scan_timing_collect()
print(json.dumps({"k": k, "N": N, "S": S, "B": B, "kernel": xp.last_scan_kernel(), "scan_ms": round(ms / n, 3),
                  "env": {e: os.environ[e] for e in os.environ if e.startswith("XPIR_")}}))
