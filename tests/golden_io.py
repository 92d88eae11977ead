"""Loaders for the committed golden fixtures (tests/golden/)."""

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_json(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def load_npz_groups(name):
    z = np.load(os.path.join(GOLDEN, name))
    out = {}
    for key in z.files:
        grp, field = key.split("/", 1)
        out.setdefault(grp, {})[field] = z[key]
    return out


def meta():
    return load_json("meta.json")


def vascular_small_text():
    with open(os.path.join(GOLDEN, "vascular_small.graph")) as fh:
        return fh.read()
