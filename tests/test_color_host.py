"""Colour-transfer host logic on CPU: value types, validation, the seeded
test-data generator (reference fixtures from tests/golden/make_golden_color.py)."""

import numpy as np
import pytest
from conftest import golden

from paper_2605_00837_b200 import color as CT


def test_make_rgb_image_clamps():
    img = CT.make_rgb_image(1, 2, np.array([[1.5, -0.2, 0.5], [0.0, 1.0, 0.25]]))
    assert img.pixels.max() <= 1.0 and img.pixels.min() >= 0.0
    assert img.pixels.shape == (2, 3)


def test_make_rgb_image_shape_validation():
    with pytest.raises(ValueError):
        CT.make_rgb_image(2, 2, np.zeros((3, 3)))


def test_sample_count_validation():
    image = CT.make_rgb_image(4, 4, np.zeros((16, 3)))
    with pytest.raises(ValueError):
        CT.color_transfer(image, image, sample_count=0, eps=0.05, seed=0)
    with pytest.raises(ValueError):
        CT.color_transfer(image, image, sample_count=17, eps=0.05, seed=0)


def test_generate_rigid_pair_matches_reference():
    G = golden("rigid_pairs")
    X, Y, perm = CT.generate_rigid_pair(50, 3, 0.3, (0.1, 0.2, 0.3), 0.01, 9)
    np.testing.assert_array_equal(X, G["X"])
    np.testing.assert_array_equal(Y, G["Y"])
    np.testing.assert_array_equal(perm, G["perm"])
    X2, Y2, perm2 = CT.generate_rigid_pair(40, 2, -0.7, (0.5, -0.25), 0.0, 4)
    np.testing.assert_array_equal(Y2, G["Y2"])
    np.testing.assert_array_equal(perm2, G["perm2"])


def test_generate_rigid_pair_validation():
    with pytest.raises(ValueError):
        CT.generate_rigid_pair(5, 4, 0.0, (0, 0, 0, 0), 0.0, 0)
    with pytest.raises(ValueError):
        CT.generate_rigid_pair(5, 2, 0.0, (0, 0), -1.0, 0)
    with pytest.raises(Exception):
        CT.generate_rigid_pair(5, 2, 0.0, (0, 0, 0), 0.0, 0)
