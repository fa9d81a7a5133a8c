"""Model documents for the harness: token grammar + shape resolution.

Mirrors the reference's model.hpp so tests and bench.py can describe the stock models
without the reference tree (which does not exist on the GPU box):
  parse_token (model.hpp:162-183), parse_atom (:124-160), resolve_model (:190-296),
  make_model (:299-315), parse_model (:317-337), needs_bn_route (:73-76).
The resolved layers are handed to the C ABI as btnn_layer_spec records.
"""
from __future__ import annotations

import ctypes as C
import json
import math
from dataclasses import dataclass, field

from . import capi


class ModelError(ValueError):
    """invalid_input (grammar) or validation_error (shapes), by .code."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


@dataclass
class Layer:
    kind: int = capi.BIT_CONV
    kh: int = 0
    kw: int = 0
    out_channels: int = 0
    stride: int = 1
    pad: int = 0
    window: int = 0
    pool_stride: int = 0
    units: int = 0
    in_h: int = 0
    in_w: int = 0
    in_channels: int = 0
    out_h: int = 0
    out_w: int = 0
    residual_out: bool = False
    residual_in: bool = False
    shortcut_from: int = -1


@dataclass
class Model:
    name: str
    in_h: int
    in_w: int
    in_c: int
    classes: int
    epsilon: float = 1e-5
    layers: list = field(default_factory=list)
    shortcuts: list = field(default_factory=list)

    # -- C ABI view -------------------------------------------------------------------
    def c_spec(self) -> capi.ModelSpec:
        arr = (capi.LayerSpec * len(self.layers))()
        for i, l in enumerate(self.layers):
            arr[i] = capi.LayerSpec(l.kind, l.kh, l.kw, l.out_channels, l.stride, l.pad, l.window, l.pool_stride,
                                    l.units, l.in_h, l.in_w, l.in_channels, l.out_h, l.out_w, int(l.residual_out),
                                    int(l.residual_in), l.shortcut_from)
        self._c_layers = arr  # keep alive
        self._c_name = self.name.encode()
        return capi.ModelSpec(self._c_name, self.in_h, self.in_w, self.in_c, self.classes, self.epsilon, arr,
                              len(self.layers))

    def bit_macs_per_image(self) -> tuple[int, int]:
        """(bit MACs, f64 MACs) per image, border taps counted as full (bench.hpp:290-292)."""
        bits = f64 = 0
        for l in self.layers:
            if l.kind == capi.FIRST_CONV_BWN:
                f64 += l.out_h * l.out_w * l.out_channels * l.in_channels * l.kh * l.kw
            elif l.kind == capi.BIT_CONV:
                bits += l.out_h * l.out_w * l.out_channels * l.in_channels * l.kh * l.kw
            elif l.kind in (capi.BIT_FC, capi.LAST_FC):
                bits += l.in_channels * l.units
        return bits, f64


def needs_bn_route(l: Layer) -> bool:
    """model.hpp:73-76."""
    return l.kind in (capi.FIRST_CONV_BWN, capi.LAST_FC) or l.residual_in or l.residual_out


def _split_top(s: str, sep: str) -> list[str]:
    parts, cur, depth = [], "", 0
    for ch in s:
        if ch == "(":
            depth += 1
        if ch == ")":
            depth -= 1
        if depth < 0:
            raise ModelError(capi.BTNN_INVALID_INPUT, f"model: unbalanced parens in '{s}'")
        if ch == sep and depth == 0:
            parts.append(cur)
            cur = ""
        else:
            cur += ch
    if depth != 0:
        raise ModelError(capi.BTNN_INVALID_INPUT, f"model: unbalanced parens in '{s}'")
    parts.append(cur)
    return parts


def _fully_parenthesized(s: str) -> bool:
    if len(s) < 2 or s[0] != "(" or s[-1] != ")":
        return False
    depth = 0
    for i, ch in enumerate(s):
        depth += ch == "("
        depth -= ch == ")"
        if depth == 0:
            return i == len(s) - 1
    return False


def _uint(s: str, tok: str) -> int:
    if not s or not s.isdigit():
        raise ModelError(capi.BTNN_INVALID_INPUT, f"model: bad token '{tok}'")
    return int(s)


def _parse_atom(tok: str, out: list) -> None:
    l = Layer()
    if len(tok) > 2 and tok.endswith("FC"):
        l.kind = capi.BIT_FC
        l.units = _uint(tok[:-2], tok)
        if l.units == 0:
            raise ModelError(capi.BTNN_INVALID_INPUT, f"model: zero units in '{tok}'")
        out.append(l)
        return
    if len(tok) > 1 and (tok[0] == "P" or (len(tok) > 2 and tok[:2] == "MP")):
        k = _uint(tok[2:] if tok[0] == "M" else tok[1:], tok)
        if k == 0:
            raise ModelError(capi.BTNN_INVALID_INPUT, f"model: zero pool window in '{tok}'")
        l.kind, l.window, l.pool_stride = capi.OR_POOL, k, k
        out.append(l)
        return
    c = tok.find("C")
    if c > 0:
        l.kind = capi.BIT_CONV
        l.out_channels = _uint(tok[:c], tok)
        rest = tok[c + 1:]
        if "/" in rest:
            rest, st = rest.split("/", 1)
            l.stride = _uint(st, tok)
        l.kh = l.kw = _uint(rest, tok)
        if l.out_channels == 0 or l.kh == 0 or l.stride == 0:
            raise ModelError(capi.BTNN_INVALID_INPUT, f"model: bad token '{tok}'")
        l.pad = l.kh // 2
        out.append(l)
        return
    raise ModelError(capi.BTNN_INVALID_INPUT, f"model: bad token '{tok}'")


def parse_token(tok: str, out: list) -> None:
    if not tok:
        raise ModelError(capi.BTNN_INVALID_INPUT, "model: empty token")
    parts = _split_top(tok, "-")
    if len(parts) > 1:
        for p in parts:
            parse_token(p, out)
        return
    i = 0
    while i < len(tok) and tok[i].isdigit():
        i += 1
    if 0 < i < len(tok) and tok[i] == "x":
        n = _uint(tok[:i], tok)
        if n == 0:
            raise ModelError(capi.BTNN_INVALID_INPUT, f"model: zero repeat in '{tok}'")
        for _ in range(n):
            parse_token(tok[i + 1:], out)
        return
    if _fully_parenthesized(tok):
        parse_token(tok[1:-1], out)
        return
    _parse_atom(tok, out)


def _label(m: Model, i: int) -> str:
    names = {0: "first_conv", 1: "bit_conv", 2: "or_pool", 3: "bit_fc", 4: "last_fc"}
    return f"layer {i} ({names[m.layers[i].kind]})"


def resolve_model(m: Model) -> None:
    """model.hpp:190-296."""
    V = capi.BTNN_VALIDATION_ERROR
    if not (m.in_h and m.in_w and m.in_c):
        raise ModelError(V, f"model '{m.name}': zero input dimension")
    if m.classes < 2:
        raise ModelError(V, f"model '{m.name}': need at least 2 classes")
    if not (m.epsilon > 0.0) or not math.isfinite(m.epsilon):
        raise ModelError(V, f"model '{m.name}': epsilon must be positive and finite")
    if not m.layers:
        raise ModelError(V, f"model '{m.name}': no layers")
    if m.layers[0].kind == capi.BIT_CONV:
        m.layers[0].kind = capi.FIRST_CONV_BWN
    elif m.layers[0].kind != capi.BIT_FC:
        raise ModelError(V, f"model '{m.name}': first layer must be conv or fc")
    m.layers.append(Layer(kind=capi.LAST_FC, units=m.classes))
    h, w, c = m.in_h, m.in_w, m.in_c
    fc_seen = False
    for i, l in enumerate(m.layers):
        l.in_h, l.in_w, l.in_channels = h, w, c
        if l.kind in (capi.FIRST_CONV_BWN, capi.BIT_CONV):
            if fc_seen:
                raise ModelError(V, f"{_label(m, i)}: conv after fc layers")
            if h + 2 * l.pad < l.kh:
                raise ModelError(V, f"{_label(m, i)}: conv: input shorter than kernel")
            if w + 2 * l.pad < l.kw:
                raise ModelError(V, f"{_label(m, i)}: conv: input narrower than kernel")
            l.out_h = (h + 2 * l.pad - l.kh) // l.stride + 1
            l.out_w = (w + 2 * l.pad - l.kw) // l.stride + 1
            h, w, c = l.out_h, l.out_w, l.out_channels
        elif l.kind == capi.OR_POOL:
            if fc_seen:
                raise ModelError(V, f"{_label(m, i)}: pool after fc layers")
            if h < l.window or w < l.window or (h - l.window) % l.pool_stride or (w - l.window) % l.pool_stride:
                raise ModelError(V, f"{_label(m, i)}: window {l.window}/{l.pool_stride} does not cover {h}x{w} exactly")
            l.out_h = (h - l.window) // l.pool_stride + 1
            l.out_w = (w - l.window) // l.pool_stride + 1
            l.out_channels = c
            h, w = l.out_h, l.out_w
        else:
            if not fc_seen:
                l.in_channels = h * w * c
                fc_seen = True
            else:
                l.in_channels = c
            l.out_h = l.out_w = 1
            h = w = 1
            c = l.units
    used_to = [False] * len(m.layers)
    for (fr, to) in m.shortcuts:
        if fr >= len(m.layers) or to >= len(m.layers):
            raise ModelError(V, f"model '{m.name}': shortcut index out of range")
        if fr >= to:
            raise ModelError(V, f"model '{m.name}': shortcut must go forward ({fr} -> {to})")
        a, b = m.layers[fr], m.layers[to]
        if a.kind not in (capi.FIRST_CONV_BWN, capi.BIT_CONV) or b.kind != capi.BIT_CONV:
            raise ModelError(V, f"model '{m.name}': shortcut {fr} -> {to} must connect conv layers")
        if used_to[to]:
            raise ModelError(V, f"{_label(m, to)}: multiple incoming shortcuts")
        used_to[to] = True
        same = a.out_h == b.out_h and a.out_w == b.out_w
        halved = a.out_h == 2 * b.out_h and a.out_w == 2 * b.out_w
        if not same and not halved:
            raise ModelError(V, f"{_label(m, to)}: shortcut spatial dims do not reach")
        if a.out_channels > b.out_channels:
            raise ModelError(V, f"{_label(m, to)}: shortcut would drop channels")
        a.residual_out = True
        b.residual_in = True
        b.shortcut_from = fr


def make_model(name: str, tokens: str, in_h: int, in_w: int, in_c: int, classes: int, shortcuts=(),
               epsilon: float = 1e-5) -> Model:
    """model.hpp:299-315."""
    m = Model(name, in_h, in_w, in_c, classes, epsilon, [], [tuple(s) for s in shortcuts])
    parse_token(tokens, m.layers)
    resolve_model(m)
    return m


def parse_model(doc: dict | str) -> Model:
    """model.hpp:317-343 (JSON document)."""
    j = json.loads(doc) if isinstance(doc, str) else doc
    try:
        m = Model(j["name"], int(j["input"]["height"]), int(j["input"]["width"]), int(j["input"]["channels"]),
                  int(j["classes"]), float(j.get("epsilon", 1e-5)), [],
                  [(int(s["from"]), int(s["to"])) for s in j.get("shortcuts", [])])
        for tok in j["layers"]:
            parse_token(tok, m.layers)
    except (KeyError, TypeError) as e:
        raise ModelError(capi.BTNN_INVALID_INPUT, f"model: bad json: {e}") from e
    resolve_model(m)
    return m


# The stock structures of the reference (proj/models/*.json, Table 6 of the paper),
# restated so the GPU box needs no reference tree.
STOCK = {
    "resnet18": {"name": "resnet18", "input": {"height": 224, "width": 224, "channels": 3}, "classes": 1000,
                 "layers": ["64C7/4-4x64C3-128C3/2-3x128C3-256C3/2-3x256C3-512C3/2-3x512C3-(2x512FC)"],
                 "shortcuts": [{"from": a, "to": a + 2} for a in range(0, 16, 2)]},
    "alexnet": {"name": "alexnet", "input": {"height": 224, "width": 224, "channels": 3}, "classes": 1000,
                "layers": ["(128C11/4)-P2-(256C5)-P2-(3x256C3)-P2-(3x4096FC)"]},
    "cifar-vgg": {"name": "cifar-vgg", "input": {"height": 32, "width": 32, "channels": 3}, "classes": 10,
                  "layers": ["(2x128C3)-MP2-(2x256C3)-MP2-(2x512C3)-MP2-(3x1024FC)"]},
    "mnist-mlp": {"name": "mnist-mlp", "input": {"height": 28, "width": 28, "channels": 1}, "classes": 10,
                  "layers": ["1024FC-1024FC-1024FC-1024FC"]},
    "cifar-resnet14": {"name": "cifar-resnet14", "input": {"height": 32, "width": 32, "channels": 3}, "classes": 10,
                       "layers": ["128C3/2-4x128C3-256C3/2-3x256C3-512C3/2-3x512C3-(2x512FC)"],
                       "shortcuts": [{"from": a, "to": a + 2} for a in range(0, 12, 2)]},
    "vgg16": {"name": "vgg16", "input": {"height": 224, "width": 224, "channels": 3}, "classes": 1000,
              "layers": ["(2x64C3)-P2-(2x128C3)-P2-(3x256C3)-P2-2x(3x512C3-P2)-(3x4096FC)"]},
}


def stock_model(name: str, height: int | None = None, width: int | None = None) -> Model:
    doc = json.loads(json.dumps(STOCK[name]))
    if height:
        doc["input"]["height"] = height
    if width:
        doc["input"]["width"] = width
    return parse_model(doc)
