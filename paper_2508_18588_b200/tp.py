"""Tensor parallelism over a GPU pair (configs[4]: Qwen2.5-32B shape, TP = 2 inside a rollout worker).

Megatron-style split (model.tp_local_config / Weights(tp_rank, tp_size)): QKV and gate/up are column-parallel
(each GPU owns half the q / kv heads and half the FFN), O and down are row-parallel (each GPU's GEMM produces
an fp32 partial of the full [rows, d] output).  The all-reduce of those partials is not an NCCL call: each
GPU's O / down GEMM writes its partial straight into a symmetric-memory buffer (mapped on both GPUs over
NVLink), a peer-memory barrier kernel (hm_tp_barrier) orders the two GPUs, and the next RMSNorm reads both
partials in place -- local from HBM, the peer's over NVLink -- summing y0 + y1 in the same order on both GPUs
(hm_rmsnorm_residual_bf16 with the default bf16 residual stream, hm_rmsnorm_residual2 with fp32), so the
replicated residual stream stays bit-identical across the pair.  Two buffers
alternate (O -> buffer 0, down -> buffer 1), so one barrier per all-reduce is enough: a GPU cannot overwrite
a buffer before its peer has passed the barrier that follows the peer's read of it.

Everything else (drafting, acceptance, attention over the GPU's own kv heads, the replicated LM head) runs
identically on both GPUs from identical inputs, inside the same captured CUDA graph.
"""

from __future__ import annotations


class TensorParallel:
    """Symmetric buffers + barrier state of one GPU of a TP pair (process group `group`, two ranks)."""

    def __init__(self, group, max_rows: int, d_model: int, device, dtype=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        self.size = dist.get_world_size(group)
        if self.size != 2:
            raise ValueError("TensorParallel supports tensor-parallel pairs (tp = 2)")
        self.rank = dist.get_rank(group)
        self.peer = 1 - self.rank
        self.device = torch.device(device)
        dtype = dtype or torch.bfloat16            # the forward's residual dtype (bf16 or fp32 partials)
        n = max_rows * d_model
        tail = 256 // torch.tensor([], dtype=dtype).element_size()   # 256 bytes of flag words
        # one symmetric allocation: [2 partial buffers of max_rows x d][flag words]
        self.buf = symm_mem.empty(2 * n + tail, dtype=dtype, device=self.device)
        self.buf.zero_()
        name = group.group_name if hasattr(group, "group_name") else dist.group.WORLD.group_name
        self.handle = symm_mem.rendezvous(self.buf, name)
        peer_buf = self.handle.get_buffer(self.peer, (2 * n + tail,), dtype)
        self.y = [self.buf[i * n:(i + 1) * n].view(max_rows, d_model) for i in range(2)]
        self.y_peer = [peer_buf[i * n:(i + 1) * n].view(max_rows, d_model) for i in range(2)]
        flags = self.buf[2 * n:].view(torch.int32)
        self.my_flag = flags[0:1]                   # written by the peer
        self.peer_flag = peer_buf[2 * n:].view(torch.int32)[0:1]
        self.gen = torch.zeros(1, dtype=torch.int32, device=self.device)   # local generation counter
        torch.cuda.synchronize(self.device)
        dist.barrier(group=group)

    def barrier(self, stream):
        from .model import check, lib
        check(lib().hm_tp_barrier(self.my_flag.data_ptr(), self.peer_flag.data_ptr(), self.gen.data_ptr(),
                                  stream.cuda_stream))
