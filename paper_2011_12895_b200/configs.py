"""The BASELINE.json workloads (SURVEY.md section 8 / Appendix C interpretations).

"B" counts segments and "T" is unroll_len (learner.cpp:108-109, replay_mem.cpp:40),
so one learner step consumes B*T frames per shard.  ``batch_size`` is per shard,
exactly as the reference's ``HyperParams::batch_size`` (learner.cpp:108).
"""
from dataclasses import dataclass, field


@dataclass(frozen=True)
class Config:
    name: str
    algo: str                 # "ppo" | "vtrace" | "ppo_vtrace"
    obs_dim: int
    n_actions: int
    hidden: tuple
    unroll_len: int           # T
    batch_size: int           # B segments per shard
    obs_kind: str = "gauss"   # "gauss" (N(0,1) rounded to f32) | "binary" (Bernoulli(0.1) planes)
    optimizer: str = "adam"
    seed: int = 1000
    note: str = ""

    @property
    def frames(self):
        return self.unroll_len * self.batch_size

    def flops_per_frame(self):
        """2*sum(in*out) fwd + 2*sum(in*out) dW + 2*sum_{l>=2}(in*out) dX, heads included
        (SURVEY.md section 8(d))."""
        dims = [self.obs_dim, *self.hidden]
        layers = [(dims[i], dims[i + 1]) for i in range(len(dims) - 1)]
        layers.append((dims[-1], self.n_actions + 1))
        mac = sum(i * o for i, o in layers)
        dx = sum(i * o for i, o in layers[1:])
        return 2 * mac + 2 * mac + 2 * dx


CONFIGS = {
    "C1": Config("C1", "ppo", 64, 6, (256, 256), 32, 64, seed=1001,
                 note="PPO, MLP 64-256-256-(6,1), GAE, T=32 B=64"),
    "C2": Config("C2", "vtrace", 64, 6, (512, 512), 80, 256, seed=1002,
                 note="V-trace, MLP 64-512-512-(6,1), T=80 B=256 (obs 64 assumed)"),
    "C3": Config("C3", "ppo", 1936, 6, (256, 256), 32, 4096, obs_kind="binary", seed=1003,
                 note="Pommerman-shaped obs 11x11x16 binary planes, PPO, T=32 B=4096 per shard"),
    "C4": Config("C4", "infer", 64, 6, (1024, 1024), 1, 65536, seed=1004,
                 note="InferenceServer batched forward, 65,536 obs, MLP 64-1024-1024-(6,1)"),
    "C5": Config("C5", "ppo_vtrace", 64, 6, (2048, 2048, 2048, 2048), 64, 2048, seed=1005,
                 note="4x2048 trunk, PPO surrogate over V-trace targets, T=64, B=16384 over "
                      "8 GPUs = 2048 segments per learner shard"),
}
