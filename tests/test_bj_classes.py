"""Host logic of the class-shared block-Jacobi inverses (solver.py
_block_classes / class_tiles): exact grouping of bit-identical blocks and
the element tiles of ldg_bj_apply_tiles.  CPU only."""

import numpy as np
import torch

from paper_2205_07824_b200.solver import _block_classes, class_tiles


def test_block_classes_groups_bit_identical_blocks():
    rng = np.random.default_rng(0)
    proto = rng.normal(size=(5, 6, 6))
    which = rng.integers(0, 5, size=400)
    mats = torch.as_tensor(proto[which].copy())
    cls, reps = _block_classes(mats)
    assert reps.numel() == 5
    assert torch.equal(mats[reps[cls]], mats)
    # same class <=> same prototype
    c = cls.numpy()
    for a in range(5):
        assert len(set(c[which == a])) == 1


def test_block_classes_declines_distinct_or_perturbed_blocks():
    rng = np.random.default_rng(1)
    mats = torch.as_tensor(rng.normal(size=(300, 4, 4)))
    assert _block_classes(mats) is None                      # every block distinct
    proto = rng.normal(size=(4, 4))
    m = np.repeat(proto[None], 300, axis=0)
    m[7, 2, 3] = np.nextafter(m[7, 2, 3], 10.0)               # one ulp apart: own class
    cls, reps = _block_classes(torch.as_tensor(m))
    assert reps.numel() == 2 and int((cls == cls[7]).sum()) == 1


def test_class_tiles_cover_every_element_once():
    rng = np.random.default_rng(2)
    classes = torch.as_tensor(rng.integers(0, 7, size=1000))
    E = 16
    tcls, tel = class_tiles(classes, 7, E)
    tel = tel.numpy().reshape(-1, E)
    assert tel.shape[0] == tcls.numel()
    seen = tel[tel >= 0]
    assert np.array_equal(np.sort(seen), np.arange(1000))
    for t in range(tel.shape[0]):
        els = tel[t][tel[t] >= 0]
        assert np.all(classes.numpy()[els] == int(tcls[t]))
        assert np.all(np.diff(els) > 0)
