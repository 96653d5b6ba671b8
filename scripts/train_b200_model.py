"""Train the B200 format selector with the REFERENCE's own, unchanged code.

Dev-time only (needs /root/reference, like tests/golden/make_golden.py):
reads the record and feature files scripts/b200_labels.py wrote on the GPU
box -- in spmvkit's file formats, parsed here by spmvkit's own
read_records / read_features -- and runs spmvkit.model.assemble_training_set,
cross_validate (k = 5, 3 repeats, with the per-format runtimes for the
performance ratio) and train_tree + save_model on all samples.

    python scripts/train_b200_model.py [--src gpurun_out]
    python scripts/train_b200_model.py --src paper_1805_11938_b200/data   # regenerate from the shipped records

Writes
    paper_1805_11938_b200/data/b200_selector.model   the shipped model (spmvkit-model v1 text)
    paper_1805_11938_b200/data/b200_records.txt      the B200 measurements it was trained on
    paper_1805_11938_b200/data/b200_features.txt     the GPU-extracted features
    tests/golden/b200_selector_predictions.json      spmvkit.predict per training matrix (pins our loader + predict)
    profiles/r02_b200_selector.md                    cross-validation report
"""

from __future__ import annotations

import argparse
import json
import shutil
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/pkg/src")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--src", default=str(ROOT / "gpurun_out"))
    ap.add_argument("--max-depth", type=int, default=8)
    ap.add_argument("--min-leaf", type=int, default=3)
    args = ap.parse_args()
    sys.path.insert(0, str(REF))
    import spmvkit  # noqa: F401  (the reference, unmodified)
    from spmvkit import bench as rbench, features as rfeat, model as rmodel
    from spmvkit.formats import FormatTag

    src = Path(args.src)
    records = rbench.read_records(src / "b200_records.txt")
    feats = rfeat.read_features(src / "b200_features.txt")
    labels = rbench.best_labels(records)
    times = rbench.times_by_matrix(records)
    samples, _, problems = rmodel.assemble_training_set(labels, feats)
    assert not problems, problems[:5]
    cv = rmodel.cross_validate(samples, k=5, seed=0, repeats=3, times=times, max_depth=args.max_depth,
                               min_samples_leaf=args.min_leaf)
    model = rmodel.train_tree(samples, args.max_depth, args.min_leaf)
    data = ROOT / "paper_1805_11938_b200" / "data"
    data.mkdir(exist_ok=True)
    rmodel.save_model(model, data / "b200_selector.model")
    if src.resolve() != data.resolve():  # --src paper_1805_11938_b200/data regenerates the model from the shipped files
        shutil.copy(src / "b200_records.txt", data / "b200_records.txt")
        shutil.copy(src / "b200_features.txt", data / "b200_features.txt")
    preds = {s.matrix_id: rmodel.predict(model, s.features).value for s in samples}
    (ROOT / "tests" / "golden" / "b200_selector_predictions.json").write_text(
        json.dumps({"labels": {k: v.value for k, v in labels.items()}, "predictions": preds}, indent=0, sort_keys=True))

    # baselines: always the single most frequent label / always each fixed format
    classes = list(FormatTag)
    hist = {t.value: sum(1 for s in samples if s.label is t) for t in classes}

    def ratio_of(choice):  # mean over matrices of best time / chosen format's time
        r = []
        for s in samples:
            per = times[s.matrix_id]
            got = per.get(choice(s))
            r.append(min(per.values()) / got if got else 0.0)
        return float(np.mean(r))

    fixed = {t.value: ratio_of(lambda s, t=t: t) for t in classes}
    train_ratio = ratio_of(lambda s: rmodel.predict(model, s.features))
    train_acc = float(np.mean([preds[s.matrix_id] == s.label.value for s in samples]))
    fam = {}
    corpus = src / "b200_corpus.jsonl"
    if not corpus.exists():
        corpus = ROOT / "profiles" / "r02_b200_corpus.jsonl"
    if corpus.exists():
        for line in corpus.read_text().splitlines():
            m = json.loads(line)
            fam.setdefault(m["family"], {}).setdefault(m["best"], 0)
            fam[m["family"]][m["best"]] += 1
    lines = [
        "# B200 format selector: spmvkit's decision tree trained on B200 labels",
        "",
        f"Corpus: {len(samples)} synthetic matrices (scripts/b200_labels.py), every format timed on one B200 by",
        "`harness.bench_corpus` (CI stopping rule of the reference, CUDA-event clock, hot cache; CSR5 omega 32 sigma 16,",
        "SELL C 32 sigma 1024, grid limit 2^28 cells).  Trained here by the reference's unchanged `train_tree`",
        f"(max_depth {args.max_depth}, min_samples_leaf {args.min_leaf}); `cross_validate` k = 5, 3 repeats, seed 0.",
        "",
        f"* best-format labels: {hist}",
        f"* cross-validated accuracy: **{cv.accuracy:.3f}** (folds {min(cv.fold_accuracies):.2f}-{max(cv.fold_accuracies):.2f})",
        f"* cross-validated performance ratio (mean best time / predicted format's time): **{cv.mean_perf_ratio:.3f}**",
        f"* on the training set: accuracy {train_acc:.3f}, performance ratio {train_ratio:.3f}; tree of {len(model.nodes)} nodes",
        "* performance ratio of always choosing one format: " + ", ".join(f"{k} {v:.3f}" for k, v in fixed.items()),
        "",
        "Confusion (rows = measured best, columns = predicted; order " + ", ".join(t.value for t in classes) + "):",
        "",
        "```",
        str(cv.confusion),
        "```",
        "",
        "Best format per family: " + "; ".join(f"{k}: {v}" for k, v in sorted(fam.items())),
        "",
    ]
    (ROOT / "profiles" / "r02_b200_selector.md").write_text("\n".join(lines))
    print("\n".join(lines))


if __name__ == "__main__":
    main()
