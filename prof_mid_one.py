"""One scan (1 GiB store, S = 4096) at batch B (argv[1]) with kernel argv[2] for ncu."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2001_08250_b200 as xp  # noqa: E402

B = int(sys.argv[1])
k = int(sys.argv[2])
S = 4096
N = (1 << 30) // S
st = xp.Store(N, S)
st.fill_keystream(bytes(32), 0)
q = torch.randint(0, 256, (B, N // 8), dtype=torch.uint8, device='cuda')
out = torch.empty((B, S), dtype=torch.uint8, device='cuda')
xp.set_scan_opts(k)
for _ in range(3):
    st.answer_batch_dev(q, N // 8, B, out, stream=torch.cuda.current_stream())
torch.cuda.synchronize()
print("ok", xp.last_scan_kernel())
