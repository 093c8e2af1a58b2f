"""Generate tests/golden/cancer_rows.npz from the reference's shipped dataset
(run HERE, where /root/reference exists; the GPU box only reads the .npz).

Restates the reference trainer's featurisation (TypeScript, not runnable in
this image: no node):
  * mulberry32 PRNG and Fisher-Yates shuffle  — trainer/src/rng.ts:5-30
  * 70/30 seeded split (seed 7)                 — trainer/src/dataset.ts:45-50, main.ts:21-30
  * three equal-width bins per feature, cut points from metrics.json
    "bin_cuts" (training split only), boundary -> lower bin, one-hot +-1
                                                 — trainer/src/dataset.ts:53-89
  * labels 1 = malignant -> +1, else -1        — trainer/src/dataset.ts:91-93
The fixture holds the 569 binned rows as stored-binary bits (0/1 for -1/+1),
the +-1 labels and the split.  tests/test_cancer.py pins the restatement: the
shipped model's oracle_eval accuracy on these rows must equal metrics.json's
train and test accuracy exactly.
"""

import json
import os

import numpy as np

REF = "/root/reference/pkg/trainer"
HERE = os.path.dirname(os.path.abspath(__file__))


def mulberry32(seed):
    state = seed & 0xFFFFFFFF

    def imul(a, b):
        return (a * b) & 0xFFFFFFFF

    def rng():
        nonlocal state
        state = (state + 0x6D2B79F5) & 0xFFFFFFFF
        t = state
        t = imul(t ^ (t >> 15), t | 1)
        t ^= (t + imul(t ^ (t >> 7), t | 61)) & 0xFFFFFFFF
        return ((t ^ (t >> 14)) & 0xFFFFFFFF) / 4294967296.0

    return rng


def shuffle(items, rng):
    for i in range(len(items) - 1, 0, -1):
        j = int(rng() * (i + 1))
        items[i], items[j] = items[j], items[i]
    return items


def main():
    lines = open(os.path.join(REF, "data", "cancer.csv")).read().strip().split("\n")
    header = lines[0].split(",")
    rows, labels = [], []
    for line in lines[1:]:
        cells = line.split(",")
        assert len(cells) == len(header)
        rows.append([float(c) for c in cells[:-1]])
        labels.append(float(cells[-1]))
    metrics = json.load(open(os.path.join(REF, "out", "metrics.json")))
    seed = int(metrics["seed"])
    order = shuffle(list(range(len(rows))), mulberry32(seed))
    cut = int(np.floor(len(rows) * 0.7 + 0.5))  # Math.round for positive values
    train, test = order[:cut], order[cut:]
    cuts = [(float(a), float(b)) for a, b in metrics["bin_cuts"]]
    bits = np.zeros((len(rows), 3 * len(cuts)), np.uint8)
    for r, row in enumerate(rows):
        for f, v in enumerate(row):
            hot = 0 if v <= cuts[f][0] else (1 if v <= cuts[f][1] else 2)
            bits[r, 3 * f + hot] = 1
    y = np.array([1 if lab == 1 else -1 for lab in labels], np.int8)
    np.savez_compressed(os.path.join(HERE, "cancer_rows.npz"), bits=bits, labels=y,
                        train=np.array(train, np.int32), test=np.array(test, np.int32),
                        accuracy_train=metrics["accuracy"]["train"], accuracy_test=metrics["accuracy"]["test"])
    print(f"{len(rows)} rows, {bits.shape[1]} bits, train {len(train)}, test {len(test)}")


if __name__ == "__main__":
    main()
