"""Test-side workload helpers: cached generator calls plus the config-3 normals that
BASELINE.json configs[2] asks for ("normals from oracle PCA over 10-NN")."""
import functools

import numpy as np

import gen
import oracle


@functools.lru_cache(maxsize=None)
def c1():
    return gen.c1_sphere()


@functools.lru_cache(maxsize=None)
def c2(n=1 << 20, m=1 << 20):
    return gen.c2_uniform(n, m)


@functools.lru_cache(maxsize=None)
def c3():
    w = gen.c3_depth()
    nrm, _ = oracle.pca_normals(w.target, 10, view=(0.0, 0.0, 0.0))
    w.target_normals = nrm
    return w


@functools.lru_cache(maxsize=None)
def c4(metric="point_to_plane", rings=64, az=31250):
    return gen.c4_lidar(metric, rings, az)


@functools.lru_cache(maxsize=None)
def c5(logn):
    return gen.c5_patches(logn)


_trees = {}


def oracle_tree(w):
    k = (w.name, w.n)
    if k not in _trees:
        _trees[k] = oracle.KDTree(w.target)
    return _trees[k]


def rot_angle(R):
    """rotation angle of R, accurate near 0 (atan2 of the skew and symmetric parts)"""
    R = np.asarray(R, np.float64)
    s = 0.5 * np.linalg.norm([R[2, 1] - R[1, 2], R[0, 2] - R[2, 0], R[1, 0] - R[0, 1]])
    c = 0.5 * (np.trace(R) - 1.0)
    return float(np.arctan2(s, c))
