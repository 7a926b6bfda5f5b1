"""The paper's model hooks: ``swap_conv2d`` and ``swap_backend``.

* ``swap_conv2d(module, algos)`` replaces, in place, every ``torch.nn.Conv2d`` of
  ``module`` with a slim ``nn.Module`` (``Conv2D``) whose forward calls the selected
  ai3 algorithm.
* ``swap_backend(module, {"conv2d": algos})`` returns an ``ai3.Model`` built from a
  symbolic trace of ``module``: the traced graph, with every
  conv2d bound to its selected algorithm.

Selectors (Listing 2 :148-152):
  * ``str``           -- that algorithm for every conv layer;
  * ``list[str]``     -- by occurrence index among the Conv2d modules in trace order;
                         an index past the end means "default";
  * ``callable``      -- called with the original ``nn.Conv2d``, returns a name.
Special names: "default" (= "guess": the framework picks),
"torch" (keep PyTorch's module; ``swap_conv2d`` only).

Algorithm/hyperparameter conflicts raise ``UnsupportedConfiguration`` at swap
time; shape-dependent errors (kernel larger than the padded
input) surface at the first forward.  ``guess`` is resolved per input shape at the
first forward and cached with the prepared weights.
"""
from __future__ import annotations

from typing import Callable, Mapping, Sequence, Union

import torch
from torch import nn

from . import _lib
from .conv import ConvPlan, UnknownAlgorithm, UnsupportedConfiguration, conv2d, layout_of, resolve

Selector = Union[str, Sequence[str], Callable[[nn.Conv2d], str]]

_KEEP = ("torch", "keep")


def _conv_params(m: nn.Conv2d):
    if m.padding_mode != "zeros":
        raise UnsupportedConfiguration(f"{m}: padding_mode={m.padding_mode!r} is not supported (zeros only)")
    pad = m.padding
    if isinstance(pad, str):
        if pad == "valid":
            pad = (0, 0)
        else:  # "same": symmetric only when every dilated kernel extent is odd
            ph = m.dilation[0] * (m.kernel_size[0] - 1)
            pw = m.dilation[1] * (m.kernel_size[1] - 1)
            if ph % 2 or pw % 2:
                raise UnsupportedConfiguration(f"{m}: padding='same' would be asymmetric")
            pad = (ph // 2, pw // 2)
    return tuple(m.stride), tuple(pad), tuple(m.dilation), m.groups


def _validate(m: nn.Conv2d, algorithm: str, name: str = ""):
    """Swap-time check of the algorithm against the layer's hyperparameters."""
    aid, custom = resolve(algorithm)  # raises UnknownAlgorithm
    stride, pad, dil, groups = _conv_params(m)
    if custom is not None:
        return custom  # what a user algorithm supports is its own business
    K, Cg, R, S = m.weight.shape
    C = Cg * groups
    # shape-independent constraints only: probe with an input just large enough
    H = dil[0] * (R - 1) + 1
    W = dil[1] * (S - 1) + 1
    lib = _lib.load()
    prm = _lib.params(K, (R, S), stride, pad, dil, groups, m.bias is not None)
    dt = _lib.BF16 if m.weight.dtype == torch.bfloat16 else _lib.F32
    st = lib.ai3_conv2d_supported(prm, _lib.shape4((1, C, H, W)), dt, _lib.MATH_STRICT, aid)
    if st == _lib.ERR_UNSUPPORTED:
        raise UnsupportedConfiguration(f"layer {name or m}: {_lib.last_error()}")
    if st == _lib.ERR_UNKNOWN_ALGORITHM:
        raise UnknownAlgorithm(_lib.last_error())
    return None


class Conv2D(nn.Module):
    """Slim replacement for ``nn.Conv2d`` whose forward runs the selected ai3 algorithm
    (PAPER.md:178).  Shares the original module's weight/bias parameters.

    One prepared plan is cached per (shape, dtype, memory format, device); it is
    rebuilt if the weights change in place (``_version`` bump).
    """

    def __init__(self, orig: nn.Conv2d, algorithm: str = "default", math: str = "strict", name: str = ""):
        super().__init__()
        self.custom = _validate(orig, algorithm, name)  # resolved registered name, or None
        self.weight = orig.weight
        self.bias = orig.bias
        self.in_channels, self.out_channels = orig.in_channels, orig.out_channels
        self.kernel_size = orig.kernel_size
        self.stride, self.padding, self.dilation, self.groups = _conv_params(orig)
        self.algorithm = algorithm
        self.math = math
        self.layer_name = name
        self._plans = {}

    def extra_repr(self):
        return (f"{self.in_channels}, {self.out_channels}, kernel_size={tuple(self.kernel_size)}, "
                f"stride={self.stride}, padding={self.padding}, algorithm={self.algorithm!r}")

    def plan_for(self, x: torch.Tensor) -> ConvPlan:
        lay = layout_of(x)
        wv = self.weight._version, None if self.bias is None else self.bias._version
        key = (tuple(x.shape), x.dtype, lay, x.device)
        ent = self._plans.get(key)
        if ent is None or ent[0] != wv:
            plan = ConvPlan(self.weight, self.bias, x.shape, self.stride, self.padding, self.dilation, self.groups,
                            self.algorithm, self.math, in_layout=lay, dtype=x.dtype)
            ent = (wv, plan)
            self._plans[key] = ent
        return ent[1]

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if not x.is_cuda:
            raise ValueError("ai3.Conv2D runs on CUDA tensors only (there is no CPU path)")
        if not (x.is_contiguous() or x.is_contiguous(memory_format=torch.channels_last)):
            x = x.contiguous()
        if self.custom is not None:  # user algorithm: one ai3_conv2d_custom call per forward
            return conv2d(x, self.weight, self.bias, self.stride, self.padding, self.dilation, self.groups,
                          self.custom, self.math)
        return self.plan_for(x)(x)


def _resolve(selector: Selector, module: nn.Conv2d, index: int) -> str:
    if isinstance(selector, str):
        return selector
    if callable(selector):
        name = selector(module)
        if not isinstance(name, str):
            raise UnknownAlgorithm(f"selector returned {name!r}, expected an algorithm name")
        return name
    seq = list(selector)
    return seq[index] if index < len(seq) else "default"


def _traced_conv_order(module: nn.Module):
    """Qualified names of the Conv2d modules in the order a symbolic pass reaches them
    (torch.fx.symbolic_trace); module registration order if tracing fails."""
    try:
        gm = torch.fx.symbolic_trace(module)
        mods = dict(module.named_modules())
        order = []
        for node in gm.graph.nodes:
            if node.op == "call_module" and isinstance(mods.get(node.target), nn.Conv2d):
                if node.target not in order:
                    order.append(node.target)
        # convs never reached by the trace keep registration order after the traced ones
        for n, m in module.named_modules():
            if isinstance(m, nn.Conv2d) and n not in order:
                order.append(n)
        return order
    except Exception:
        return [n for n, m in module.named_modules() if isinstance(m, nn.Conv2d)]


def _set_submodule(root: nn.Module, qualname: str, new: nn.Module):
    parent_name, _, attr = qualname.rpartition(".")
    parent = root.get_submodule(parent_name) if parent_name else root
    setattr(parent, attr, new)


def swap_conv2d(module: nn.Module, algos: Selector = "default", math: str = "strict") -> nn.Module:
    """Replace every ``nn.Conv2d`` of ``module`` in place.

    Returns ``module`` for convenience.  Layers whose selector says "torch" are kept.
    """
    order = _traced_conv_order(module)
    swaps = []
    for i, qn in enumerate(order):
        conv = module.get_submodule(qn)
        name = _resolve(algos, conv, i)
        if name in _KEEP:
            continue
        swaps.append((qn, Conv2D(conv, name, math, qn)))  # validates at swap time
    for qn, new in swaps:
        _set_submodule(module, qn, new)
    return module


class Model(nn.Module):
    """Result of ``swap_backend``: the traced graph of the original
    module with each conv2d bound to its selected ai3 algorithm.

    Scope note: ai3 kernels cover conv2d, the hot path; the other
    traced operations (pooling, activations, linear, flatten) still execute through
    the graph as PyTorch ops -- the all-ai3 operator set is SURVEY §8 row f1.
    """

    def __init__(self, graph_module: nn.Module, layers):
        super().__init__()
        self.graph_module = graph_module
        self.layers = layers  # [(qualname, algorithm)] in trace order

    def forward(self, *args, **kwargs):
        return self.graph_module(*args, **kwargs)


def swap_backend(module: nn.Module, algos: Mapping[str, Selector] | None = None, math: str = "strict") -> Model:
    """Build an ``ai3.Model`` from ``module``.  ``algos`` maps an
    operation name to a selector; only "conv2d" is algorithm-selectable."""
    algos = dict(algos or {})
    unknown = set(algos) - {"conv2d"}
    if unknown:
        raise UnknownAlgorithm(f"no selectable operation named {sorted(unknown)} (supported: conv2d)")
    sel = algos.get("conv2d", "default")
    import copy
    gm = torch.fx.symbolic_trace(copy.deepcopy(module))
    order = _traced_conv_order(gm)
    layers = []
    for i, qn in enumerate(order):
        conv = gm.get_submodule(qn)
        name = _resolve(sel, conv, i)
        if name in _KEEP:
            raise UnsupportedConfiguration("'torch' is only valid for swap_conv2d (PAPER.md:170)")
        _set_submodule(gm, qn, Conv2D(conv, name, math, qn))
        layers.append((qn, name))
    gm.recompile()
    return Model(gm, layers)
