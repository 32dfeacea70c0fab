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
        self.lo_hi = np.asarray(lo_hi, np.float32)
        self.n_global = int(n_global)
        e2 = float(sum((float(lo_hi[d + m]) - float(lo_hi[m])) ** 2 for m in range(d)))
        tot = self.n_global * e2 * (1.0 + 2.0 ** -20)
        self.sse_scale = math.ldexp(1.0, 62 - math.frexp(tot)[1]) if tot > 0 else 1.0

    def step(self):
        a = oracle.assign(self.points, self.C.astype(np.float64))
        changed = self.n if self.labels is None else int((a.labels != self.labels).sum())
        self.labels = a.labels
        S = np.zeros((self.k, self.d), np.int64)
        np.add.at(S, self.labels, self.q)
        cnt = np.bincount(self.labels, minlength=self.k).astype(np.int64)
        sse_t = int(np.rint(a.best.sum() * self.sse_scale))
        part = np.concatenate([S.ravel(), cnt, [changed, sse_t]]).astype(np.int64)
        return torch.from_numpy(part)

    def apply(self, part, tol, want_done):
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
        """Eq. 1 of the shard as an integer multiple of 2^-s3 (per-point rounding, the bound B =
        squared diagonal of the global box united with the centroids' box, as km.h states),
        returned as 48-bit limbs."""
        d = self.d
        P64 = self.points.astype(np.float64)
        C64 = self.C.astype(np.float64)
        lo = np.minimum(self.lo_hi[:d], self.C.min(0)).astype(np.float64)
        hi = np.maximum(self.lo_hi[d:], self.C.max(0)).astype(np.float64)
        b = 0.0
        for m in range(d):
            b += (hi[m] - lo[m]) ** 2
        tot = self.n_global * b * (1.0 + 2.0 ** -20)
        self.s3 = 126 - math.frexp(tot)[1] if tot > 0 else 0
        t = P64[:, 0] - C64[self.labels, 0]
        D = t * t
        for m in range(1, d):
            t = P64[:, m] - C64[self.labels, m]
            D = D + t * t
        v = np.rint(D * math.ldexp(1.0, self.s3))
        total = sum(int(x) for x in v)
        m48 = (1 << 48) - 1
        limbs = np.array([total & m48, (total >> 48) & m48, total >> 96], np.int64)
        return torch.from_numpy(self.C.copy()), torch.from_numpy(self.labels.copy()), self.it, limbs

    def sse(self, limbs_sum):
        l = [int(x) for x in np.asarray(limbs_sum)]
        total = l[0] + (l[1] << 48) + (l[2] << 96)
        hi, lo = total >> 64, total & ((1 << 64) - 1)
        return (float(hi) * 2.0 ** 64 + float(lo)) * math.ldexp(1.0, -self.s3)
