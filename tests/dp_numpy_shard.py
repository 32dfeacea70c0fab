"""Test-only CPU stand-in for LibkmShard (same interface), used to exercise the data-parallel
host logic of paper_2412_02244_b200.dp with gloo on CPU.  Assignment comes from the FP64
oracle (the exact labels libkm certifies); sums use the same 64-bit fixed point and the same
refine formula as libkm's finalize, so sharded and unsharded runs must agree bit for bit."""
import math

import numpy as np
import torch

import oracle


class NumpyShard:
    def __init__(self, points: np.ndarray, k: int):
        self.points = np.ascontiguousarray(points, np.float32)
        self.n, self.d = self.points.shape
        self.k = k

    def bbox(self):
        return np.concatenate([self.points.min(0), self.points.max(0)]).astype(np.float32)

    def begin(self, init, lo_hi, n_global, max_iter):
        d = self.d
        init = init.cpu().numpy() if hasattr(init, "cpu") else np.asarray(init)
        self.C = np.asarray(init, np.float32).copy()
        nb = int(n_global).bit_length()
        self.o = lo_hi[:d].astype(np.float64)
        self.scale = np.zeros(d)
        self.inv = np.zeros(d)
        for m in range(d):
            ext = float(lo_hi[d + m]) - float(lo_hi[m])
            s = 61 - nb - math.frexp(ext)[1] if ext > 0 else 0
            self.scale[m] = math.ldexp(1.0, s)
            self.inv[m] = math.ldexp(1.0, -s)
        self.q = np.rint((self.points.astype(np.float64) - self.o) * self.scale).astype(np.int64)
        self.labels = None
        self.it = 0
        self.done = False

    def step(self):
        a = oracle.assign(self.points, self.C.astype(np.float64))
        changed = self.n if self.labels is None else int((a.labels != self.labels).sum())
        self.labels = a.labels
        S = np.zeros((self.k, self.d), np.int64)
        np.add.at(S, self.labels, self.q)
        cnt = np.bincount(self.labels, minlength=self.k).astype(np.int64)
        part = np.concatenate([S.ravel(), cnt, [changed]]).astype(np.int64)
        return torch.from_numpy(part), torch.tensor([a.best.sum()], dtype=torch.float64)

    def apply(self, part, sse, tol, want_done):
        kd = self.k * self.d
        p = part.numpy()
        S = p[:kd].reshape(self.k, self.d).astype(np.float64)
        cnt = p[kd:kd + self.k]
        changed = int(p[kd + self.k])
        old = self.C.astype(np.float64)
        new = self.C.copy()
        nz = cnt > 0
        mean = self.o + (S[nz] / cnt[nz, None].astype(np.float64)) * self.inv
        new[nz] = mean.astype(np.float32)
        drift = np.sqrt(((new.astype(np.float64) - old) ** 2).sum(1)).max()
        self.C = new
        t = self.it
        self.it += 1
        if tol >= 0 and (drift <= tol or (t >= 1 and changed == 0)):
            self.done = True
        return self.it, self.done if want_done else None

    def end(self):
        sse = oracle.sse(self.points, self.labels, self.C.astype(np.float64))
        return torch.from_numpy(self.C.copy()), torch.from_numpy(self.labels.copy()), sse, self.it
