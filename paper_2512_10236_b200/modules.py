"""Torch modules over the FiCCO ops: the callers SURVEY.md §8b adds to the reference (which has none).

Tensor/sequence parallelism as in the paper's TP/SP scenarios: activations are sequence-sharded
between the blocks, so a column-parallel layer starts with an all-gather of its input rows and a
row-parallel layer ends with a reduce-scatter of its output rows. Each direction of each layer is one
overlapped FiCCO op, and the backward pass is the adjoint op:

=========================  ======================================  =========================================
layer                      forward                                 backward (input gradient)
=========================  ======================================  =========================================
SequenceParallelColumn     Y = all_gather(X_shard) @ W^T           dX_shard = reduce_scatter(dY @ W)
  (up-projection, C2/C3')  (ops.all_gather_matmul)                 (ops.matmul_reduce_scatter)
SequenceParallelRow        Y_shard = reduce_scatter(X @ W^T)       dX = all_gather(dY_shard) @ W
  (down-projection, C3)    (ops.matmul_reduce_scatter)             (ops.all_gather_matmul)
=========================  ======================================  =========================================

Weight gradients are plain GEMMs of tensors every rank holds after the op (the gathered X of the forward
all-gather, the gathered dY of the backward all-gather): torch.matmul. ``ContextParallelScores`` wraps the
CP KV all-gather -> QK^T op (forward only: the scores feed a softmax the caller owns).

Operands are bf16 and contiguous (the ops' boundary checks raise ValueError otherwise); the schedule is
the selector's choice unless ``kind`` / ``backward_kind`` are given. A ``FiccoGroup`` is one per device
(ops.FiccoGroup.distributed(), one process per GPU).
"""
from __future__ import annotations

import math

import torch

from . import ops


class _AllGatherLinear(torch.autograd.Function):
    """Y = all_gather(X_shard) @ W^T; backward dX_shard = reduce_scatter(dY @ W), dW = dY^T @ X_all."""

    @staticmethod
    def forward(ctx, x_shard, weight, group, kind, backward_kind, comm_agent):
        y, gathered = ops.all_gather_matmul(x_shard, weight, kind=kind, group=group, return_gathered=True,
                                            comm_agent=comm_agent)
        # the gathered view lives in the group's double-buffered workspace (valid until the call after
        # next): keep a copy for the weight gradient
        ctx.save_for_backward(gathered.clone(), weight)
        ctx.group, ctx.backward_kind, ctx.comm_agent = group, backward_kind, comm_agent
        return y

    @staticmethod
    def backward(ctx, dy):
        gathered, weight = ctx.saved_tensors
        dy = dy.contiguous()
        dx = dw = None
        if ctx.needs_input_grad[0]:
            # dY [M, N] @ W [N, K] = dY @ (W^T)^T: the RS op's weight operand is W^T [K, N] (nn.Linear layout)
            dx = ops.matmul_reduce_scatter(dy, weight.t().contiguous(), kind=ctx.backward_kind, group=ctx.group)
        if ctx.needs_input_grad[1]:
            dw = dy.t() @ gathered
        return dx, dw, None, None, None, None


class _LinearReduceScatter(torch.autograd.Function):
    """Y_shard = reduce_scatter(X @ W^T); backward dX = all_gather(dY_shard) @ W, dW = all_gather(dY)^T @ X."""

    @staticmethod
    def forward(ctx, x, weight, group, kind, backward_kind, comm_agent):
        y = ops.matmul_reduce_scatter(x, weight, kind=kind, group=group, comm_agent=comm_agent)
        ctx.save_for_backward(x, weight)
        ctx.group, ctx.backward_kind = group, backward_kind
        return y

    @staticmethod
    def backward(ctx, dy_shard):
        x, weight = ctx.saved_tensors
        # dX [M, K] = all_gather(dY_shard) [M, N] @ W [N, K]: the AG op's weight operand is W^T [K, N]
        dx, dy_all = ops.all_gather_matmul(dy_shard.contiguous(), weight.t().contiguous(), kind=ctx.backward_kind,
                                           group=ctx.group, return_gathered=True)
        dw = dy_all.t() @ x if ctx.needs_input_grad[1] else None
        return (dx if ctx.needs_input_grad[0] else None), dw, None, None, None, None


class SequenceParallelColumnLinear(torch.nn.Module):
    """Column-parallel linear with a sequence-sharded input: [R, in] per rank -> [G*R, out_local].

    ``weight`` [out_local, in] is this rank's column block (nn.Linear layout), e.g. the gate||up
    projection of a TP MLP (C2: Llama-3-8B, out_local = 2 * 14336 / G)."""

    def __init__(self, in_features: int, out_local: int, group: "ops.FiccoGroup", kind=None, backward_kind=None,
                 comm_agent=None, device=None):
        super().__init__()
        self.group, self.kind, self.backward_kind, self.comm_agent = group, kind, backward_kind, comm_agent
        w = torch.empty(out_local, in_features, dtype=torch.bfloat16, device=device)
        torch.nn.init.normal_(w, std=1.0 / math.sqrt(in_features))
        self.weight = torch.nn.Parameter(w)

    def forward(self, x_shard: torch.Tensor) -> torch.Tensor:
        return _AllGatherLinear.apply(x_shard, self.weight, self.group, self.kind, self.backward_kind,
                                      self.comm_agent)


class SequenceParallelRowLinear(torch.nn.Module):
    """Row-parallel linear with a sequence-sharded output: [M, in_local] per rank -> [M/G, out].

    ``weight`` [out, in_local] is this rank's row block (nn.Linear layout), e.g. the down projection of a
    TP MLP (C3: Llama-3-70B, in_local = 28672 / G)."""

    def __init__(self, in_local: int, out_features: int, group: "ops.FiccoGroup", kind=None, backward_kind=None,
                 comm_agent=None, device=None):
        super().__init__()
        self.group, self.kind, self.backward_kind, self.comm_agent = group, kind, backward_kind, comm_agent
        w = torch.empty(out_features, in_local, dtype=torch.bfloat16, device=device)
        torch.nn.init.normal_(w, std=1.0 / math.sqrt(in_local * group.world))
        self.weight = torch.nn.Parameter(w)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return _LinearReduceScatter.apply(x, self.weight, self.group, self.kind, self.backward_kind,
                                          self.comm_agent)


class ContextParallelScores(torch.nn.Module):
    """Context-parallel attention scores: S = scale * Q @ all_gather(K_shard)^T (one head, forward only)."""

    def __init__(self, group: "ops.FiccoGroup", kind=None, scale: float | None = None, comm_agent=None):
        super().__init__()
        self.group, self.kind, self.scale, self.comm_agent = group, kind, scale, comm_agent

    def forward(self, q: torch.Tensor, k_shard: torch.Tensor) -> torch.Tensor:
        return ops.cp_kv_all_gather_qk(q, k_shard, kind=self.kind, scale=self.scale, group=self.group,
                                       comm_agent=self.comm_agent)


__all__ = ["SequenceParallelColumnLinear", "SequenceParallelRowLinear", "ContextParallelScores"]
