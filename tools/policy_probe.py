"""C4 InfServer forward timing probe (device-resident batch, CUDA events on the policy
stream).  Env switches of the library apply (TLG_POLICY_I8, TLG_I8X2_BN).  Test tool."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_12895_b200 as tlg  # noqa: E402

B = int(os.environ.get("PROBE_BATCH", "65536"))
D, A, H = 64, 6, (1024, 1024)
pol = tlg.Policy("mlp", D, A, H, max_batch=B)
n_p = D * H[0] + H[0] + H[0] * H[1] + H[1] + (A + 1) * H[1] + A + 1
pol.set_params(tlg.synth.init_params_f32(n_p, 0.05, seed=1).astype(np.float64))
ob = torch.from_numpy(tlg.synth.make_obs(B, D, seed=1)).cuda()
lg = torch.empty(B, A, device="cuda")
pr = torch.empty_like(lg)
v = torch.empty(B, device="cuda")
s = torch.cuda.ExternalStream(pol.stream())
reps = int(os.environ.get("PROBE_REPS", "20"))
for _ in range(3):
    pol.forward_device(ob, lg, pr, v)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(reps):
    pol.forward_device(ob, lg, pr, v)
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"policy_probe B={B} env I8={os.environ.get('TLG_POLICY_I8')} BN={os.environ.get('TLG_I8X2_BN')}"
      f" ms/batch={ms:.4f} Mactions/s={B / ms / 1e3:.1f}")
