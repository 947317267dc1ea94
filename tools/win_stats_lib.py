"""Shared helper of the tuning scripts: nearest object row per pixel (numpy)."""
import numpy as np


def nearest_rows(feat):
    H, W = feat.shape
    INF = 1 << 20
    up = np.full((H, W), -INF, np.int64)
    last = np.full(W, -INF, np.int64)
    for i in range(H):
        last = np.where(feat[i], i, last); up[i] = last
    dn = np.full((H, W), INF, np.int64)
    nxt = np.full(W, INF, np.int64)
    for i in range(H - 1, -1, -1):
        nxt = np.where(feat[i], i, nxt); dn[i] = nxt
    ii = np.arange(H)[:, None]
    nr = np.where(ii - up <= dn - ii, up, dn)
    return np.where(np.abs(nr) >= INF // 2, -1, nr)
