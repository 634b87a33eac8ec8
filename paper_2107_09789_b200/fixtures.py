"""Benchmark fixture graphs in the reference IR.

The reference ships no model graphs; these rebuild the three networks the
BASELINE configs name, with random weights drawn from one
``np.random.default_rng(seed)`` stream in node-creation order:
Conv He-normal N(0, 2/(k*k*c)), Linear N(0, 1/c), BatchNorm rows
scale U(0.5,1.5), shift N(0,0.1), mean N(0,0.1), var U(0.5,1.5).
Node ids follow creation order, which fixes topo tie-breaks and trace order.
"""

from __future__ import annotations

import numpy as np

from .ir import Graph, Node, OperatorKind, TensorShape


class _Builder:
    def __init__(self, input_shape: TensorShape, seed: int):
        self.rng = np.random.default_rng(seed)
        self.nodes: dict[int, Node] = {}
        self.input_shape = input_shape

    def _add(self, kind, attrs, weights, inputs) -> int:
        nid = len(self.nodes)
        self.nodes[nid] = Node(nid, kind, attrs, weights, list(inputs))
        return nid

    def conv(self, src: list[int], c: int, j: int, k: int, stride: int = 1, padding: int = 0) -> int:
        w = (self.rng.standard_normal((k, k, c, j)) * np.sqrt(2.0 / (k * k * c))).astype(np.float32)
        return self._add(OperatorKind.Conv2D, {"k1": k, "k2": k, "c": c, "j": j, "stride": stride,
                                               "padding": padding}, w, src)

    def linear(self, src: int, c: int, j: int) -> int:
        w = (self.rng.standard_normal((c, j)) * np.sqrt(1.0 / c)).astype(np.float32)
        return self._add(OperatorKind.Linear, {"c": c, "j": j}, w, [src])

    def bn(self, src: int, c: int) -> int:
        scale = self.rng.uniform(0.5, 1.5, c)
        shift = self.rng.normal(0.0, 0.1, c)
        mean = self.rng.normal(0.0, 0.1, c)
        var = self.rng.uniform(0.5, 1.5, c)
        return self._add(OperatorKind.BatchNorm, {}, np.stack([scale, shift, mean, var]).astype(np.float32), [src])

    def relu(self, src: int) -> int:
        return self._add(OperatorKind.ReLU, {}, None, [src])

    def pool(self, src: int, window: int, stride: int) -> int:
        return self._add(OperatorKind.MaxPool, {"window": window, "stride": stride}, None, [src])

    def add(self, srcs: list[int]) -> int:
        return self._add(OperatorKind.Add, {}, None, srcs)

    def softmax(self, src: int) -> int:
        return self._add(OperatorKind.SoftMax, {}, None, [src])

    def graph(self, out: int) -> Graph:
        return Graph(self.nodes, out, self.input_shape)


def c1c2(batch: int = 1, size: int = 56, seed: int = 0) -> Graph:
    """Config 1: C1(3->64) BN ReLU -> C2(64->128) BN ReLU -> C3(128->128) ReLU, 3x3 p1.
    C3 gives C2 a consumer so it can be widened (transforms.py:82-101)."""
    b = _Builder(TensorShape(batch, 3, size, size), seed)
    x = b.relu(b.bn(b.conv([], 3, 64, 3, 1, 1), 64))
    x = b.relu(b.bn(b.conv([x], 64, 128, 3, 1, 1), 128))
    x = b.relu(b.conv([x], 128, 128, 3, 1, 1))
    return b.graph(x)


def resnet18(batch: int = 1, size: int = 224, classes: int = 1000, seed: int = 0) -> Graph:
    """ResNet-18 in the reference IR: MaxPool w2 s2 stem pool (no pool padding,
    graph.py:195-201) and a MaxPool w7 s1 global-pool stand-in (no AvgPool op)."""
    b = _Builder(TensorShape(batch, 3, size, size), seed)
    x = b.pool(b.relu(b.bn(b.conv([], 3, 64, 7, 2, 3), 64)), 2, 2)
    cin = 64
    for stage, width in enumerate((64, 128, 256, 512)):
        for blk in range(2):
            stride = 2 if (stage > 0 and blk == 0) else 1
            y = b.relu(b.bn(b.conv([x], cin, width, 3, stride, 1), width))
            y = b.bn(b.conv([y], width, width, 3, 1, 1), width)
            if stride != 1 or cin != width:
                sc = b.bn(b.conv([x], cin, width, 1, stride, 0), width)
            else:
                sc = x
            x = b.relu(b.add([y, sc]))
            cin = width
    spatial = size // 32
    x = b.pool(x, spatial, 1)
    x = b.softmax(b.linear(x, 512, classes))
    return b.graph(x)


VGG16_CFG = (64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M", 512, 512, 512, "M")


def vgg16(batch: int = 1, size: int = 224, classes: int = 1000, seed: int = 0, hidden: int = 4096) -> Graph:
    """VGG-16 with BatchNorm: 13 x (Conv3x3 p1, BN, ReLU), 5 MaxPool w2 s2, 3 Linear."""
    b = _Builder(TensorShape(batch, 3, size, size), seed)
    x, cin, first = None, 3, True
    for item in VGG16_CFG:
        if item == "M":
            x = b.pool(x, 2, 2)
            continue
        x = b.relu(b.bn(b.conv([] if first else [x], cin, item, 3, 1, 1), item))
        cin, first = item, False
    spatial = size // 32
    x = b.relu(b.linear(x, 512 * spatial * spatial, hidden))
    x = b.relu(b.linear(x, hidden, hidden))
    x = b.softmax(b.linear(x, hidden, classes))
    return b.graph(x)


FIXTURES = {"c1c2": c1c2, "resnet18": resnet18, "vgg16": vgg16}
