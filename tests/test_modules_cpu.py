"""Host-side checks of the torch modules over the FiCCO ops (no GPU): parameter layout (nn.Linear:
[out, in] per rank's block), dtype, and that the autograd Functions return one gradient slot per
forward input (the GPU test test_modules_gpu.py runs them)."""
import inspect

import torch

from paper_2512_10236_b200 import modules, ops


def test_module_parameters_follow_the_tp_sp_layout():
    grp = ops.FiccoGroup.virtual_group(4, 1)
    col = modules.SequenceParallelColumnLinear(256, 128, grp)
    row = modules.SequenceParallelRowLinear(128, 256, grp)
    assert col.weight.shape == (128, 256) and row.weight.shape == (256, 128)
    assert col.weight.dtype == row.weight.dtype == torch.bfloat16
    assert col.weight.requires_grad and row.weight.requires_grad
    assert [n for n, _ in col.named_parameters()] == ["weight"]
    cp = modules.ContextParallelScores(grp, scale=0.125)
    assert cp.scale == 0.125 and list(cp.parameters()) == []


def test_autograd_functions_return_a_slot_per_input():
    for fn in (modules._AllGatherLinear, modules._LinearReduceScatter):
        n_in = len(inspect.signature(fn.forward).parameters) - 1  # minus ctx
        src = inspect.getsource(fn.backward)
        assert src.count("None") >= n_in - 2  # x and weight get gradients, the rest None
