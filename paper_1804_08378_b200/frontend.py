"""PyTorch front-end: find stacks in a network, run them depth-first.

PAPER.md §4 "PyTorch Front-end and API": "The frontend parses through the neural
network, groups all optimizable layers in stacks and passes these to the BrainSlug optimizer.
These are then removed from the network and replaced by a special BrainSlug layer (one per
stack) that pass the control flow to the BrainSlug scheduler whenever they are triggered."
`lst:python` shows the two-line use: ``model = brainslug.optimize(model)``.

Here the network graph comes from ``torch.fx.symbolic_trace`` and every stack is replaced by a
:class:`BrainSlugStack` module whose forward is one ``bs_execute_ex`` call through the C ABI
(include/bs.h) on the current CUDA stream -- argument marshalling only; the stack runs in
libbrainslug.so's sm_100a kernels.  There is no CPU fallback: a stack fed a CPU tensor raises.

Optimizable layers ("element-wise and pooling"):
  BatchNorm2d (inference: running statistics)  -> BATCHNORM
  ReLU / F.relu / torch.relu / Tensor.relu      -> RELU
  MaxPool2d (dilation 1, floor mode)            -> MAXPOOL
  AvgPool2d (floor mode, no divisor override)   -> AVGPOOL
  AdaptiveAvgPool2d(1) / F.adaptive_avg_pool2d(., 1): global average -> AVGPOOL over H x W
  Dropout (eval: identity)                      -> COPY
  a + b (residual add; not counted as a layer)  -> ADD (the other summand is an extra input)
  x * c (python number)                         -> SCALE
Chaining rule (Appendix A): a node joins the current stack iff it consumes the stack's last
node and that node has no other consumer (so ``torch.cat`` inputs and branch points end a
stack).  Anything else (convolutions, linear layers, concatenation, flatten) is a barrier.

Plans are shape-bound: a BrainSlugStack creates one plan per input shape on first
use and reuses it.  BatchNorm parameters are folded when that plan is created (inference only;
re-optimize after changing weights).  The paper generates code once for identical stacks
(P:L590-592); plans here are cheap, so each stack owns its own.
"""
from __future__ import annotations

import dataclasses
import operator
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch
import torch.fx as fx
import torch.nn as nn
import torch.nn.functional as F

from . import bs_execute_ex, bs_plan_create, bs_plan_query


@dataclasses.dataclass
class LayerSpec:
    """A layer description in the binding's duck-typed form (see paper_1804_08378_b200.__init__)."""
    kind: str
    kernel: Tuple[int, int] = (1, 1)
    stride: Tuple[int, int] = (1, 1)
    padding: Tuple[int, int] = (0, 0)
    count_include_pad: bool = True
    eps: float = 1e-5
    gamma: Optional[np.ndarray] = None
    beta: Optional[np.ndarray] = None
    mean: Optional[np.ndarray] = None
    var: Optional[np.ndarray] = None
    alpha: float = 1.0
    operand: int = 0
    global_pool: bool = False   # AdaptiveAvgPool2d(1): kernel = stride = input H x W at plan time
    module: Optional[nn.Module] = None   # BatchNorm2d whose statistics are read at plan time


def _pair(v) -> Tuple[int, int]:
    return (int(v[0]), int(v[1])) if isinstance(v, (tuple, list)) else (int(v), int(v))


def _is_global(out_size) -> bool:
    return out_size == 1 or tuple(out_size) in ((1, 1),)


# ----------------------------------------------------------------------------- classification
def _classify(gm: fx.GraphModule, n: fx.Node) -> Optional[Tuple[LayerSpec, fx.Node, Optional[fx.Node]]]:
    """(layer, data input node, ADD operand node) if `n` is an optimizable layer, else None."""
    if n.op == "call_module":
        m = gm.get_submodule(n.target)
        x = n.args[0] if n.args else None
        if not isinstance(x, fx.Node):
            return None
        if isinstance(m, nn.BatchNorm2d):
            if not m.track_running_stats or m.running_mean is None or m.training:
                return None
            return LayerSpec("batchnorm", eps=float(m.eps), module=m), x, None
        if isinstance(m, nn.ReLU):
            # an in-place ReLU also rewrites its input for that input's other consumers: keep
            # such a node in eager PyTorch (a stack writes a new tensor)
            if m.inplace and len(x.users) > 1:
                return None
            return LayerSpec("relu"), x, None
        if isinstance(m, nn.MaxPool2d):
            if _pair(m.dilation) != (1, 1) or m.ceil_mode or m.return_indices:
                return None
            k = _pair(m.kernel_size)
            s = _pair(m.stride if m.stride is not None else m.kernel_size)
            return LayerSpec("maxpool", kernel=k, stride=s, padding=_pair(m.padding)), x, None
        if isinstance(m, nn.AvgPool2d):
            if m.ceil_mode or m.divisor_override is not None:
                return None
            k = _pair(m.kernel_size)
            s = _pair(m.stride if m.stride is not None else m.kernel_size)
            return (LayerSpec("avgpool", kernel=k, stride=s, padding=_pair(m.padding),
                              count_include_pad=bool(m.count_include_pad)), x, None)
        if isinstance(m, nn.AdaptiveAvgPool2d):
            return (LayerSpec("avgpool", global_pool=True), x, None) if _is_global(m.output_size) else None
        if isinstance(m, nn.Dropout):
            return (LayerSpec("copy"), x, None) if not m.training else None
        return None
    if n.op == "call_function":
        if n.target in (F.relu, torch.relu) and n.args and isinstance(n.args[0], fx.Node):
            if n.kwargs.get("inplace", False) and len(n.args[0].users) > 1:
                return None
            return LayerSpec("relu"), n.args[0], None
        if n.target is F.adaptive_avg_pool2d and len(n.args) >= 2 and isinstance(n.args[0], fx.Node) \
                and _is_global(n.args[1]):
            return LayerSpec("avgpool", global_pool=True), n.args[0], None
        if n.target in (operator.add, torch.add) and len(n.args) == 2 and not n.kwargs:
            a, b = n.args
            if isinstance(a, fx.Node) and isinstance(b, fx.Node) and a is not b:
                return LayerSpec("add"), a, b   # data input resolved against the chain in find_stacks
        if n.target in (operator.mul, torch.mul) and len(n.args) == 2 and not n.kwargs:
            a, b = n.args
            if isinstance(a, fx.Node) and isinstance(b, (int, float)) and not isinstance(b, bool):
                return LayerSpec("scale", alpha=float(b)), a, None
            if isinstance(b, fx.Node) and isinstance(a, (int, float)) and not isinstance(a, bool):
                return LayerSpec("scale", alpha=float(a)), b, None
        return None
    if n.op == "call_method" and n.target == "relu" and n.args and isinstance(n.args[0], fx.Node):
        return LayerSpec("relu"), n.args[0], None
    return None


@dataclasses.dataclass
class Stack:
    """One stack found in the graph: its nodes (in order), input node and ADD operand nodes."""
    nodes: List[fx.Node]
    layers: List[LayerSpec]
    input: fx.Node
    operands: List[fx.Node]

    @property
    def n_layers(self) -> int:
        """Optimizable layers (the paper's "Opt." count; a residual ADD is not a layer)."""
        return sum(1 for L in self.layers if L.kind != "add")

    def signature(self) -> str:
        return "[" + ",".join(L.kind for L in self.layers) + "]"


def _meta(n) -> Optional[object]:
    return n.meta.get("tensor_meta") if isinstance(n, fx.Node) else None


def _shape_ok(spec: LayerSpec, n: fx.Node, x: fx.Node, opnd: Optional[fx.Node]) -> bool:
    """With shape metadata (ShapeProp over an example input): the data input must be a float32
    tensor (4-D for anything but a flat element-wise layer), and an ADD must be a same-shape,
    same-dtype residual add -- a broadcasting add stays in PyTorch."""
    mx, mn = _meta(x), _meta(n)
    if mx is None or mn is None:   # ShapeProp records tensor_meta for tensor values only
        return False
    if not hasattr(mx, "shape") or mx.dtype != torch.float32:
        return False
    if len(mx.shape) != 4 and spec.kind not in ("relu", "copy", "scale", "add"):
        return False
    if spec.kind == "add":
        mo = _meta(opnd)
        return (mo is not None and hasattr(mo, "shape") and mo.dtype == torch.float32
                and tuple(mo.shape) == tuple(mx.shape) == tuple(mn.shape))
    return True


def find_stacks(gm: fx.GraphModule) -> List[Stack]:
    """Group the optimizable nodes of `gm`'s graph into stacks (SURVEY.md Appendix A rule).
    When the graph carries shape metadata (``optimize(model, example_input)``), only float32
    tensor nodes are classified and ADDs must be same-shape residual adds."""
    stacks: List[Stack] = []
    cur: Optional[Stack] = None
    has_meta = any("tensor_meta" in n.meta for n in gm.graph.nodes)
    for n in gm.graph.nodes:
        c = _classify(gm, n)
        if c is None:
            continue
        spec, x, opnd = c
        if has_meta and not _shape_ok(spec, n, x, opnd):
            continue
        if spec.kind == "add":
            # the summand that continues the current stack is the data input, the other an operand
            a, b = x, opnd
            if cur is not None and b is cur.nodes[-1]:
                a, b = b, a
            x, opnd = a, b
        tail_ok = cur is not None and x is cur.nodes[-1] and len(cur.nodes[-1].users) == 1
        if tail_ok:
            cur.nodes.append(n)
            cur.layers.append(spec)
        else:
            cur = Stack(nodes=[n], layers=[spec], input=x, operands=[])
            stacks.append(cur)
        if spec.kind == "add":
            cur.operands.append(opnd)
            spec.operand = len(cur.operands)
    return stacks


# ----------------------------------------------------------------------------- the BrainSlug layer
class BrainSlugStack(nn.Module):
    """One stack, executed depth-first by libbrainslug.so."""

    def __init__(self, layers: Sequence[LayerSpec], name: str = ""):
        super().__init__()
        self.layers = list(layers)
        self.name = name
        self._plans: Dict[Tuple, object] = {}

    def signature(self) -> str:
        return "[" + ",".join(L.kind for L in self.layers) + "]"

    def _resolved_layers(self, shape) -> List[LayerSpec]:
        """Global pools take the H x W at their position; BN statistics are read now."""
        _, _, H, W = shape
        out = []
        for L in self.layers:
            L = dataclasses.replace(L)
            if L.kind == "batchnorm":
                m = L.module
                C = m.running_mean.numel()
                w = m.weight.detach() if m.weight is not None else torch.ones(C)
                b = m.bias.detach() if m.bias is not None else torch.zeros(C)
                L.gamma, L.beta = (w.float().cpu().numpy(), b.float().cpu().numpy())
                L.mean = m.running_mean.detach().float().cpu().numpy()
                L.var = m.running_var.detach().float().cpu().numpy()
                L.module = None
            if L.kind in ("maxpool", "avgpool"):
                if L.global_pool:
                    L.kernel, L.stride, L.padding = (H, W), (H, W), (0, 0)
                (kh, kw), (sh, sw), (ph, pw) = L.kernel, L.stride, L.padding
                H, W = (H + 2 * ph - kh) // sh + 1, (W + 2 * pw - kw) // sw + 1
            out.append(L)
        return out

    def _scalar_forward(self, x, operands):
        """A stack classified from the graph alone can receive Python numbers (e.g. ``x.shape[2] * 2``
        traced without example inputs): evaluate it with plain Python semantics -- this is graph
        bookkeeping, not tensor work, and nothing of a tensor runs here."""
        for L in self.layers:
            if L.kind == "relu":
                x = x if x > 0 else 0 * x
            elif L.kind == "copy":
                pass
            elif L.kind == "scale":
                x = x * L.alpha
            elif L.kind == "add":
                x = x + operands[L.operand - 1]
            else:
                raise TypeError(f"BrainSlugStack {self.name}: a {L.kind} layer needs a tensor, got {type(x)}")
        return x

    def _check_operands(self, x: torch.Tensor, operands) -> List[torch.Tensor]:
        """Each ADD operand must have the shape of the tensor at its layer (the C ABI reads exactly
        that many elements): broadcastable operands are expanded, anything else is an error."""
        shape = tuple(x.shape)
        N, C, H, W = shape
        want = {}
        for L in self.layers:
            if L.kind == "add":
                want[L.operand] = (N, C, H, W)
            elif L.kind in ("maxpool", "avgpool") and not L.global_pool:
                (kh, kw), (sh, sw), (ph, pw) = L.kernel, L.stride, L.padding
                H, W = (H + 2 * ph - kh) // sh + 1, (W + 2 * pw - kw) // sw + 1
            elif L.kind in ("maxpool", "avgpool"):
                H, W = 1, 1
        out = []
        for k, o in enumerate(operands, start=1):
            if not isinstance(o, torch.Tensor):
                o = torch.as_tensor(o, dtype=torch.float32, device=x.device)
            if o.device != x.device or o.dtype != torch.float32:
                raise RuntimeError(f"BrainSlugStack {self.name}: ADD operand {k} is {o.dtype} on {o.device}; "
                                   f"needs float32 on {x.device}")
            exp = want[k]
            if tuple(o.shape) != exp:
                try:
                    ok = tuple(torch.broadcast_shapes(tuple(o.shape), exp)) == exp
                except RuntimeError:
                    ok = False
                if not ok:
                    raise RuntimeError(f"BrainSlugStack {self.name}: ADD operand {k} of shape {tuple(o.shape)} "
                                       f"does not broadcast to the stack tensor {exp} at that layer")
                o = o.expand(exp)
            out.append(o.contiguous())
        return out

    def forward(self, x: torch.Tensor, *operands: torch.Tensor) -> torch.Tensor:
        if not isinstance(x, torch.Tensor):
            return self._scalar_forward(x, operands)
        if not x.is_cuda:
            raise RuntimeError(f"BrainSlugStack {self.name}: input on {x.device}; the stack runs only on "
                               "CUDA (sm_100a kernels) -- there is no CPU fallback")
        flat = x.dim() != 4 and all(L.kind in ("relu", "copy", "scale", "add") for L in self.layers)
        if x.dtype != torch.float32 or not (x.dim() == 4 or flat):
            raise RuntimeError(f"BrainSlugStack {self.name}: needs a 4-D float32 NCHW tensor, got "
                               f"{x.dtype} {tuple(x.shape)}")
        if flat:   # element-wise stack on a non-image tensor (e.g. a classifier's ReLU/Dropout)
            shape = x.shape
            flat4 = (1, 1, 1, x.numel()) if x.numel() else (0, 1, 1, 1)   # empty: an empty batch
            for k, o in enumerate(operands, start=1):
                if not isinstance(o, torch.Tensor) or o.dtype != torch.float32 or o.device != x.device:
                    raise RuntimeError(f"BrainSlugStack {self.name}: ADD operand {k} must be a float32 "
                                       f"tensor on {x.device}")
                if tuple(torch.broadcast_shapes(tuple(o.shape), tuple(shape))) != tuple(shape):
                    raise RuntimeError(f"BrainSlugStack {self.name}: ADD operand {k} of shape "
                                       f"{tuple(o.shape)} does not broadcast to {tuple(shape)}")
            y = self.forward(x.reshape(flat4), *[o.expand(shape).reshape(flat4) for o in operands])
            return y.reshape(shape)
        x = x.contiguous()
        ops = self._check_operands(x, operands)
        key = (tuple(x.shape), x.device.index)
        entry = self._plans.get(key)
        if entry is None:
            plan = bs_plan_create(self._resolved_layers(x.shape), x.shape, {"device": x.device.index})
            entry = self._plans[key] = (plan, tuple(bs_plan_query(plan)["out"]))
        plan, out_shape = entry
        out = torch.empty(out_shape, device=x.device, dtype=torch.float32)
        bs_execute_ex(plan, [x] + ops, out, torch.cuda.current_stream(x.device))
        return out

    def extra_repr(self) -> str:
        return self.signature()


def optimize(model: nn.Module, min_layers: int = 1, example_input: Optional[torch.Tensor] = None) -> fx.GraphModule:
    """``brainslug.optimize(model)`` (lst:python P:L531-543): the model with every stack of
    >= `min_layers` optimizable layers replaced by a BrainSlugStack.  `model` must be in eval
    mode (inference BatchNorm / Dropout); the result runs on CUDA.  With `example_input` the
    graph is shape-propagated first (torch.fx ShapeProp, on that tensor's device) and only
    float32 tensor nodes / same-shape residual adds join stacks; without it, classification is
    structural and each stack checks its operands at run time."""
    if model.training:
        raise ValueError("optimize() needs an eval-mode model (inference BatchNorm and Dropout)")
    gm = model if isinstance(model, fx.GraphModule) else fx.symbolic_trace(model)
    if example_input is not None:
        from torch.fx.passes.shape_prop import ShapeProp
        with torch.no_grad():
            ShapeProp(gm).propagate(example_input)
    stacks = find_stacks(gm)
    replaced: Dict[fx.Node, fx.Node] = {}   # tail of an already replaced stack -> its new node
    for i, st in enumerate(stacks):
        if st.n_layers < min_layers:
            continue
        name = f"brainslug_stack_{i}"
        gm.add_submodule(name, BrainSlugStack(st.layers, name))
        tail = st.nodes[-1]
        args = tuple(replaced.get(a, a) for a in (st.input, *st.operands))
        with gm.graph.inserting_after(tail):
            new = gm.graph.call_module(name, args=args)
        tail.replace_all_uses_with(new)
        replaced[tail] = new
        for n in reversed(st.nodes):
            gm.graph.erase_node(n)
    gm.graph.lint()
    gm.recompile()
    return gm


def summary(model: nn.Module) -> Dict[str, object]:
    """Counts of the paper's tbl:eval_detailkernel columns for `model`: optimizable layers
    ("Opt.") and stacks ("Stacks"), plus the stack signatures."""
    gm = model if isinstance(model, fx.GraphModule) else fx.symbolic_trace(model.eval())
    stacks = find_stacks(gm)
    return {"opt_layers": sum(s.n_layers for s in stacks), "stacks": len(stacks),
            "signatures": [s.signature() for s in stacks]}
