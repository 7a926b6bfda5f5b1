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
        self._last = None  # (shape, strides, dtype, device, weight / bias versions, plan) of the last call
        self._relu = False  # fused ReLU epilogue (set by swap_backend for conv -> relu pairs)
        self._pool = False  # fused 2x2 / stride-2 max pooling (set by swap_backend for conv (-> relu) -> pool)

    # changing a fusion flag invalidates the prepared plans (they carry the epilogue)
    @property
    def relu(self) -> bool:
        return self._relu

    @relu.setter
    def relu(self, v: bool):
        self._relu = bool(v)
        self._plans = {}
        self._last = None

    @property
    def pool(self) -> bool:
        return self._pool

    @pool.setter
    def pool(self, v: bool):
        self._pool = bool(v)
        self._plans = {}
        self._last = None

    def extra_repr(self):
        return (f"{self.in_channels}, {self.out_channels}, kernel_size={tuple(self.kernel_size)}, "
                f"stride={self.stride}, padding={self.padding}, algorithm={self.algorithm!r}")

    def plan_for(self, x: torch.Tensor) -> ConvPlan:
        lay = layout_of(x)
        wv = self.weight._version, None if self.bias is None else self.bias._version
        key = (tuple(x.shape), x.dtype, lay, x.device)
        ent = self._plans.get(key)
        if ent is None or ent[0] != wv:
            if self.algorithm == "benchmark":  # measure every algorithm once for this shape
                from .conv import autotune
                autotune(x, self.weight, self.bias, self.stride, self.padding, self.dilation, self.groups, self.math)
            plan = ConvPlan(self.weight, self.bias, x.shape, self.stride, self.padding, self.dilation, self.groups,
                            self.algorithm, self.math, in_layout=lay, dtype=x.dtype)
            if self.relu:
                plan.set_relu(True)
            plan.pool_fallback = False
            if self.pool:
                try:
                    plan.set_maxpool2x2(True)
                except UnsupportedConfiguration:  # this plan's kernel mode cannot pool: separate ai3 pass
                    plan.pool_fallback = True
            ent = (wv, plan)
            self._plans[key] = ent
        return ent[1]

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        # hot path: same input geometry and weight versions as the previous call -> the cached
        # plan's one C-ABI call (identical strides imply the memory format the plan was built for)
        last = self._last
        if last is not None and x.shape == last[0] and x.stride() == last[1] and x.dtype == last[2] and \
                x.device == last[3] and self.weight._version == last[4] and \
                (self.bias is None or self.bias._version == last[5]):
            return last[6].run_checked(x)
        if not x.is_cuda:
            raise ValueError("ai3.Conv2D runs on CUDA tensors only (there is no CPU path)")
        if not (x.is_contiguous() or x.is_contiguous(memory_format=torch.channels_last)):
            x = x.contiguous()
        if self.custom is not None:  # user algorithm: one ai3_conv2d_custom call per forward
            y = conv2d(x, self.weight, self.bias, self.stride, self.padding, self.dilation, self.groups,
                       self.custom, self.math)
            if self.relu:
                from .layers import relu
                y = relu(y, inplace=True)
            if self.pool:
                from .layers import max_pool2d
                y = max_pool2d(y, 2, 2)
            return y
        plan = self.plan_for(x)
        y = plan(x)
        if plan.pool_fallback:
            from .layers import max_pool2d
            y = max_pool2d(y, 2, 2)
        elif x.is_contiguous() or x.is_contiguous(memory_format=torch.channels_last):
            self._last = (x.shape, x.stride(), x.dtype, x.device, self.weight._version,
                          None if self.bias is None else self.bias._version, plan)
        return y


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
    """Result of ``swap_backend`` ("returns an object completely
    managed by the framework"): the traced graph of the original module with every
    supported module and function replaced by ai3's (conv2d with its selected algorithm,
    linear, ReLU, max / average / adaptive-average pooling, flatten).

    Activations run NHWC (channels_last) end to end: 4-D inputs are converted once at
    entry by ai3's layout kernel.  Conv -> ReLU pairs run as one kernel (fused epilogue);
    flatten -> linear reads the NHWC activation directly.  ``cuda_graph=True`` captures
    the forward per input shape in a CUDA graph after one eager warm-up call and replays
    it (static input/output buffers; the returned tensor is overwritten by the next call).
    """

    def __init__(self, graph_module: nn.Module, layers, replaced=(), kept=(), cuda_graph: bool = False):
        super().__init__()
        self.graph_module = graph_module
        self.layers = layers          # [(qualname, algorithm)] of the convolutions, in trace order
        self.replaced = list(replaced)  # [(node, ai3 op)] everything swapped
        self.kept = list(kept)          # [(node, target)] left as PyTorch (unsupported by ai3)
        self.cuda_graph = cuda_graph
        self._graphs = {}

    def _eager(self, *args):
        from .layers import to_layout
        args = tuple(to_layout(a, _lib.NHWC) if isinstance(a, torch.Tensor) and a.dim() == 4 and a.is_cuda
                     and a.is_floating_point() else a for a in args)
        return self.graph_module(*args)

    def forward(self, *args):
        if not self.cuda_graph or not all(isinstance(a, torch.Tensor) and a.is_cuda for a in args):
            return self._eager(*args)
        key = tuple((tuple(a.shape), a.dtype, a.device, a.stride()) for a in args)
        ent = self._graphs.get(key)
        if ent is None:
            out = self._eager(*args)  # warm-up: plans, weight preparation, workspaces
            torch.cuda.current_stream().synchronize()
            static_in = [a.clone() for a in args]
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                static_out = self._eager(*static_in)
            self._graphs[key] = (g, static_in, static_out)
            return out
        g, static_in, static_out = ent
        for s, a in zip(static_in, args):
            s.copy_(a)
        g.replay()
        return static_out


def _is_fn(target, *fns):
    return any(target is f for f in fns)


def swap_backend(module: nn.Module, algos: Mapping[str, Selector] | None = None, math: str = "strict",
                 cuda_graph: bool = False) -> Model:
    """Build an ``ai3.Model`` from ``module``.

    Every supported PyTorch module and function of the traced graph is replaced by ai3's
    implementation; ``algos`` maps an operation name to a selector and only "conv2d" is
    algorithm-selectable (the other operations have one implementation each).
    Operations ai3 does not implement stay PyTorch ops and are listed in ``Model.kept``.
    Dropout is the identity in the inference graph and is removed.
    """
    import copy
    import operator

    import torch.nn.functional as F

    from . import layers as L

    algos = dict(algos or {})
    unknown = set(algos) - {"conv2d"}
    if unknown:
        raise UnknownAlgorithm(f"no selectable operation named {sorted(unknown)} (supported: conv2d)")
    sel = algos.get("conv2d", "default")
    gm = torch.fx.symbolic_trace(copy.deepcopy(module).eval())
    order = _traced_conv_order(gm)
    layers, replaced, kept = [], [], []
    for i, qn in enumerate(order):
        conv = gm.get_submodule(qn)
        name = _resolve(sel, conv, i)
        if name in _KEEP:
            raise UnsupportedConfiguration("'torch' is only valid for swap_conv2d (PAPER.md:170)")
        _set_submodule(gm, qn, Conv2D(conv, name, math, qn))
        layers.append((qn, name))
        replaced.append((qn, "conv2d:" + name))

    graph = gm.graph
    mods = dict(gm.named_modules())
    for node in list(graph.nodes):
        if node.op == "call_module":
            m = mods[node.target]
            new = None
            if isinstance(m, (Conv2D, L.ReLU, L.MaxPool2D, L.AvgPool2D, L.AdaptiveAvgPool2D, L.Flatten, L.Linear)):
                continue  # already swapped (a module called more than once)
            if isinstance(m, nn.ReLU):
                new = L.ReLU()
            elif isinstance(m, nn.MaxPool2d):
                new = L.MaxPool2D(m)
            elif isinstance(m, nn.AvgPool2d):
                new = L.AvgPool2D(m)
            elif isinstance(m, nn.AdaptiveAvgPool2d):
                new = L.AdaptiveAvgPool2D(m)
            elif isinstance(m, nn.Flatten):
                new = L.Flatten(m)
            elif isinstance(m, nn.Linear):
                new = L.Linear(m, math)
            elif isinstance(m, (nn.Dropout, nn.Identity)):
                node.replace_all_uses_with(node.args[0])
                graph.erase_node(node)
                replaced.append((node.target, "identity"))
                continue
            if new is None:
                kept.append((node.target, type(m).__name__))
                continue
            _set_submodule(gm, node.target, new)
            mods[node.target] = new
            replaced.append((node.target, type(new).__name__))
        elif node.op == "call_function" or node.op == "call_method":
            t = node.target
            if node.op == "call_function" and _is_fn(t, torch.relu, F.relu, torch.relu_):
                node.target = L.relu
                node.kwargs = {k: v for k, v in node.kwargs.items() if k != "inplace"}
                if len(node.args) > 1:
                    node.args = node.args[:1]
            elif node.op == "call_function" and _is_fn(t, torch.flatten):
                node.target = L.flatten
            elif node.op == "call_function" and _is_fn(t, F.max_pool2d):
                node.target = L.max_pool2d
            elif node.op == "call_function" and _is_fn(t, F.avg_pool2d):
                node.target = L.avg_pool2d
            elif node.op == "call_function" and _is_fn(t, F.adaptive_avg_pool2d):
                node.target = L.adaptive_avg_pool2d
            elif node.op == "call_method" and t == "relu":
                node.op, node.target = "call_function", L.relu
            elif node.op == "call_function" and _is_fn(t, F.dropout):
                node.replace_all_uses_with(node.args[0])
                graph.erase_node(node)
                replaced.append((node.name, "identity"))
                continue
            elif node.op == "call_function" and t in (operator.getitem, getattr):
                continue
            else:
                kept.append((node.name, getattr(t, "__name__", str(t))))
                continue
            replaced.append((node.name, node.target.__name__))

    # fusions below change a module's behaviour, so they only apply to modules called from
    # exactly one node (a module reused at several call sites keeps its plain semantics)
    calls = {}
    for n in graph.nodes:
        if n.op == "call_module":
            calls[n.target] = calls.get(n.target, 0) + 1

    # fusion: conv2d / linear -> relu (sole consumer) runs as one kernel (fused epilogue)
    def _mod(n):
        return mods.get(n.target) if n.op == "call_module" else None

    def _is_relu(n):
        return (n.op == "call_function" and n.target is L.relu) or isinstance(_mod(n), L.ReLU)

    for node in list(graph.nodes):
        if not _is_relu(node) or not node.args or not isinstance(node.args[0], torch.fx.Node):
            continue
        src = node.args[0]
        producer = _mod(src)
        if isinstance(producer, (Conv2D, L.Linear)) and len(src.users) == 1 and not producer.relu and \
                calls.get(src.target) == 1:
            producer.relu = True
            node.replace_all_uses_with(src)
            graph.erase_node(node)
            replaced.append((src.name, "fused_relu"))

    # fusion: conv2d (-> relu) -> max_pool2d(2, 2) (sole consumer, floor mode, no padding or
    # dilation) runs as one kernel: the epilogue pools and the conv output never reaches memory
    def _is_pool2x2(n):
        m = _mod(n)
        if isinstance(m, L.MaxPool2D):
            k, st, pd, dl, ceil = m.args
        elif n.op == "call_function" and n.target is L.max_pool2d:
            names = ("kernel_size", "stride", "padding", "dilation", "ceil_mode")
            vals = dict(zip(names, list(n.args[1:]))) | {k2: v for k2, v in n.kwargs.items() if k2 in names}
            k, st, pd, dl, ceil = (vals.get("kernel_size"), vals.get("stride"), vals.get("padding", 0),
                                   vals.get("dilation", 1), vals.get("ceil_mode", False))
            if st is None:
                st = k
        else:
            return False
        two = lambda v: v in (2, (2, 2), [2, 2])  # noqa: E731
        zero = lambda v: v in (0, (0, 0), [0, 0])  # noqa: E731
        one = lambda v: v in (1, (1, 1), [1, 1])  # noqa: E731
        return two(k) and two(st) and zero(pd) and one(dl) and not ceil

    for node in list(graph.nodes):
        if not _is_pool2x2(node) or not node.args or not isinstance(node.args[0], torch.fx.Node):
            continue
        src = node.args[0]
        producer = _mod(src)
        if isinstance(producer, Conv2D) and len(src.users) == 1 and not producer.pool and \
                calls.get(src.target) == 1:
            producer.pool = True
            node.replace_all_uses_with(src)
            graph.erase_node(node)
            replaced.append((src.name, "fused_maxpool2x2"))

    # fusion: flatten(x, 1) -> linear is one convolution with an H x W kernel over x, which
    # reads the (NHWC) activation in place (layers.Linear.fused_flatten)
    for node in list(graph.nodes):
        is_flat = (node.op == "call_function" and node.target is L.flatten) or isinstance(_mod(node), L.Flatten)
        if not is_flat or len(node.users) != 1:
            continue
        user = next(iter(node.users))
        start_dim = node.args[1] if len(node.args) > 1 else node.kwargs.get("start_dim", 1)
        if isinstance(_mod(node), L.Flatten):
            start_dim = _mod(node).start_dim
        end_dim = node.args[2] if len(node.args) > 2 else node.kwargs.get("end_dim", -1)
        if isinstance(_mod(node), L.Flatten):
            end_dim = _mod(node).end_dim
        if isinstance(_mod(user), L.Linear) and start_dim == 1 and end_dim == -1 and user.args[0] is node and \
                calls.get(user.target) == 1:
            _mod(user).fused_flatten = True
            user.args = (node.args[0],) + tuple(user.args[1:])
            graph.erase_node(node)
            replaced.append((user.name, "flatten_fused"))

    graph.lint()
    gm.recompile()
    return Model(gm, layers, replaced, kept, cuda_graph)
