"""fp64 CPU oracle for the LegoDiffusion denoise-step hot path.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import this package.
The product path (paper_2604_08123_b200) never imports it and shares no code
with it.
"""
from .flux_step import (  # noqa: F401
    OracleLoRA,
    attention,
    dit_step,
    gelu_tanh,
    layer_norm,
    rms_norm,
    rope_cos_sin,
    apply_rope,
    timestep_embedding,
    weights_to_f64,
)
