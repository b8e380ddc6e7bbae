"""B200-native TFLA (Tiled Flash Linear Attention) for mLSTMexp / mLSTMsig.

The hot path (chunkwise forward / backward) runs in hand-written sm_100a
kernels behind the C ABI of ``include/tfla/tfla.h``; this package mirrors the
reference ``mlstm::`` API over it (see :mod:`paper_2503_14376_b200.mlstm`).
"""
from . import _ffi  # noqa: F401
from .mlstm import (  # noqa: F401
    BlockConfig,
    ChunkStates,
    ChunkwiseForward,
    ChunkwiseGates,
    CudaError,
    Dims,
    GeometryError,
    Gradients,
    MemoryState,
    NumericError,
    ParameterError,
    RecurrentTrace,
    SavedStats,
    SequenceInputs,
    StatePass,
    TfLaDkResult,
    TfLaDqResult,
    Variant,
    apply_gate_softcap,
    assemble_gate_grads,
    backward_state_pass,
    block_needs_mask,
    chunkwise_backward,
    chunkwise_forward,
    chunkwise_forward_frozen,
    chunkwise_forward_gated,
    chunkwise_gates,
    output_norm_gate,
    recurrent_step,
    kv_block_count,
    run_recurrent,
    stab,
    state_recurrence,
    tfla_backward,
    tfla_backward_dk,
    tfla_backward_dq,
    tfla_backward_dv,
    tfla_forward,
    tfla_forward_parallel,
    train_step_host,
)
