"""Format selection at deployment time (mirrors the deployment half of
spmvkit.model: ``predict``, ``select_format``, ``load_model``).

Reference: /root/reference/pkg/src/spmvkit/model.py:216-223 (predict),
:305-319 (select_format), :322-430 (model text format).  Tree training and
cross-validation are offline CPU code and out of scope;
models trained by the reference load here unchanged, and reference
``DecisionTreeModel`` objects are accepted directly (duck-typed).

``select_format`` = GPU feature extraction (8 scalars come back to the host),
host tree descent, GPU conversion.
"""

from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .features import FEATURE_NAMES, FeatureVector, ScalingParams, apply_scaling, extract_features
from .formats import FormatMatrix, FormatTag, convert

__all__ = ["B200_SELECTOR_PARAMS", "DecisionTreeModel", "ModelIOError", "TreeNode", "default_model", "load_model",
           "predict", "select_format", "select_format_b200"]

N_FEATURES = len(FEATURE_NAMES)
N_CLASSES = len(FormatTag)


class ModelIOError(ValueError):
    """A model file could not be parsed or fails structural validation."""


@dataclass
class TreeNode:
    """Internal node (feature >= 0) or leaf (feature == -1)."""

    feature: int = -1
    threshold: float = 0.0
    left: int = -1
    right: int = -1
    label: FormatTag | None = None
    counts: tuple[int, ...] = ()

    @property
    def is_leaf(self) -> bool:
        return self.feature < 0


@dataclass
class DecisionTreeModel:
    nodes: list[TreeNode]
    max_depth: int
    min_samples_leaf: int
    scaling: ScalingParams


def predict(model, f: FeatureVector) -> FormatTag:
    """Scale (clamped) and descend the tree (model.py:216-223)."""
    vec = apply_scaling(f, model.scaling)
    node = model.nodes[0]
    while not node.is_leaf:
        node = model.nodes[node.left if vec[node.feature] <= node.threshold else node.right]
    return FormatTag(node.label.value if hasattr(node.label, "value") else node.label)


def select_format(
    a,
    model,
    *,
    omega: int = 4,
    sigma: int = 16,
    sell_c: int = 4,
    sell_sigma: int = 0,
) -> tuple[FormatTag, FormatMatrix]:
    """Extract features, predict the format, convert (model.py:305-319)."""
    tag = predict(model, extract_features(a))
    return tag, convert(tag, a, omega=omega, sigma=sigma, sell_c=sell_c, sell_sigma=sell_sigma)


def _float(tok: str) -> float:
    # The reference writer formats scale extremes with repr(); under numpy 2
    # that yields "np.float64(25.0)" (model.py:338-339), which the reference
    # reader cannot parse back.  Accept both spellings.
    if tok.startswith("np.float64(") and tok.endswith(")"):
        tok = tok[len("np.float64("):-1]
    return float(tok)


def _parse_line(toks: list[str], nodes: dict, mins: np.ndarray, maxs: np.ndarray) -> None:
    kind = toks[0]
    if kind == "node" and len(toks) == 7 and toks[2] == "split":
        nodes[int(toks[1])] = TreeNode(feature=int(toks[3]), threshold=float(toks[4]), left=int(toks[5]),
                                       right=int(toks[6]))
    elif kind == "leaf" and len(toks) == 3 + N_CLASSES:
        nodes[int(toks[1])] = TreeNode(label=FormatTag(toks[2]), counts=tuple(int(c) for c in toks[3:]))
    elif kind == "scale" and len(toks) == 4:
        f = int(toks[1])
        if not 0 <= f < N_FEATURES:
            raise ValueError(f"feature index {f}")
        mins[f] = _float(toks[2])
        maxs[f] = _float(toks[3])
    else:
        raise ValueError("unrecognized line")


def _ordered_tree(nodes: dict[int, TreeNode]) -> list[TreeNode]:
    if 0 not in nodes:
        raise ModelIOError("model has no root node 0")
    missing = [i for i in range(len(nodes)) if i not in nodes]
    if missing:
        raise ModelIOError(f"node ids are not contiguous: missing {missing[0]}")
    tree = [nodes[i] for i in range(len(nodes))]
    visited: set[int] = set()
    todo = [0]
    while todo:
        i = todo.pop()
        if i in visited:
            raise ModelIOError(f"node {i} is reachable twice")
        visited.add(i)
        if not tree[i].is_leaf:
            for child in (tree[i].left, tree[i].right):
                if not 0 <= child < len(tree):
                    raise ModelIOError(f"node {i} points at missing child {child}")
                todo.append(child)
    if len(visited) != len(tree):
        raise ModelIOError("model contains unreachable nodes")
    return tree


def load_model(source) -> DecisionTreeModel:
    """Read the reference's ``spmvkit-model v1`` text format (model.py:322-430)."""
    text = source.read() if hasattr(source, "read") else Path(source).read_text()
    lines = [ln for ln in text.splitlines() if ln.strip()]
    if not lines:
        raise ModelIOError("empty model file")
    head = lines[0].split()
    ok = len(head) == 6 and head[:3] == ["spmvkit-model", "v1", "max_depth"] and head[4] == "min_samples_leaf"
    try:
        if not ok:
            raise ValueError
        max_depth, min_leaf = int(head[3]), int(head[5])
    except ValueError:
        raise ModelIOError(f"bad model header {lines[0]!r}") from None
    nodes: dict[int, TreeNode] = {}
    mins = np.full(N_FEATURES, np.nan)
    maxs = np.full(N_FEATURES, np.nan)
    for line in lines[1:]:
        try:
            _parse_line(line.split(), nodes, mins, maxs)
        except ValueError as exc:
            raise ModelIOError(f"bad model line {line!r}: {exc}") from None
    if np.isnan(mins).any() or np.isnan(maxs).any():
        raise ModelIOError("model file is missing scale lines")
    for node in nodes.values():
        if not node.is_leaf and not 0 <= node.feature < N_FEATURES:
            raise ModelIOError(f"split on unknown feature {node.feature}")
    return DecisionTreeModel(_ordered_tree(nodes), max_depth, min_leaf, ScalingParams(mins, maxs))


# The shipped B200 selector: the reference's decision tree (its unchanged
# train_tree, scripts/train_b200_model.py) fitted to best-format labels
# measured on a B200 for a 222-matrix synthetic corpus
# (scripts/b200_labels.py; records and features in data/).  Cross-validated
# with the reference's cross_validate: accuracy 0.64, and the predicted
# format runs at 0.97 of the best format's speed on average (always-CSR:
# 0.85) -- profiles/r02_b200_selector.md.  The labels were measured with these
# conversion parameters, so select_format_b200 converts with them.
B200_SELECTOR_PARAMS = dict(omega=32, sigma=16, sell_c=32, sell_sigma=1024)
_DATA = Path(__file__).resolve().with_name("data")
_default_model: DecisionTreeModel | None = None


def default_model() -> DecisionTreeModel:
    """The shipped B200 selector (data/b200_selector.model)."""
    global _default_model
    if _default_model is None:
        _default_model = load_model(_DATA / "b200_selector.model")
    return _default_model


def select_format_b200(a, *, max_cells: int = 1 << 28) -> tuple[FormatTag, FormatMatrix]:
    """``select_format`` with the shipped B200 model and the conversion
    parameters its labels were measured with.  If the predicted format cannot
    hold the matrix (ConversionError: the padded grid is too large), CSR5 is
    used, as the reference's callers fall back to CSR-family formats."""
    from ._lib import ConversionError

    tag = predict(default_model(), extract_features(a))
    try:
        return tag, convert(tag, a, max_cells=max_cells, **B200_SELECTOR_PARAMS)
    except ConversionError:
        return FormatTag.CSR5, convert(FormatTag.CSR5, a, **B200_SELECTOR_PARAMS)


# GPU-tuned conversion parameters of the measured selector (the bench's
# candidates): wide CSR5 tiles and SELL slices.
MEASURED_CANDIDATES = {
    FormatTag.CSR: {},
    FormatTag.CSR5: dict(omega=32, sigma=16),
    FormatTag.ELL: {},
    FormatTag.SELL: dict(sell_c=32, sell_sigma=1024),
    FormatTag.HYB: {},
}


def select_format_measured(a, formats=None, *, params=None, reps: int = 10, warmup: int = 3):
    """Measured-time selector (what the multi-GPU driver
    does per shard): convert to each candidate format on the GPU, time its
    SpMV with CUDA events on an all-ones x, keep the fastest.  Formats whose
    conversion fails (ConversionError, out of memory) are skipped.  Returns
    (tag, converted matrix, {tag: seconds per SpMV}); ties go to FormatTag
    declaration order."""
    import torch

    from ._lib import ConversionError
    from .kernels import bind

    tags = [FormatTag(f) for f in formats] if formats else list(FormatTag)
    params = params or MEASURED_CANDIDATES
    dev = a.device  # a COO or a CSR matrix
    x = torch.ones(a.n_cols, dtype=torch.float64, device=dev)
    y = torch.empty(a.n_rows, dtype=torch.float64, device=dev)
    times, best = {}, None
    for tag in tags:
        try:
            m = convert(tag, a, **params.get(tag, {}))
        except (ConversionError, MemoryError):
            continue
        call = bind(tag, m, x, y)  # prepared launch: the timing is the kernels', not Python dispatch
        for _ in range(warmup):
            call()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            call()
        e1.record()
        e1.synchronize()
        times[tag] = e0.elapsed_time(e1) / 1e3 / reps
        if best is None or times[tag] < times[best[0]]:
            best = (tag, m)
    if best is None:
        raise ConversionError("no candidate format converted")
    return best[0], best[1], times
