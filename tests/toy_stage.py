"""CPU stand-in of one library stage (tests only): the same per-call contract as
libsdv2 (R2 entries from the library's host control plane, parity-double-buffered act
and ring packets, per-(block, lane) state) with toy float64 arithmetic, so the
pipeline transport can be exercised with gloo on CPU."""
import numpy as np
import torch

from paper_2511_07399_b200.sdv2 import HostControl


class _IO:
    def __init__(self, d):
        self.__dict__.update(d)


class ToyStage:
    def __init__(self, n, K, rank, b0, b1, L=4, d=8, CTHW=6):
        self.n, self.K, self.rank, self.b0, self.b1 = n, K, rank, b0, b1
        self.L, self.d, self.CTHW = L, d, CTHW
        self.ctl = HostControl(1, 1, 2, n, K, rank, 1000, 0.95)
        self.ctl.set_prompt_mean([1.0], 0)
        self.pk = n * L * d + 2 * n + n * CTHW          # packet: x, sig, sign, lat (float64)
        self.ws = torch.zeros(8 * (4 * self.pk + 4 * max(1, n - 1) * CTHW), dtype=torch.uint8)
        f = self.ws.view(torch.float64)
        o = 0
        self.act = {}
        for io in ("in", "out"):
            for p in (0, 1):
                self.act[(io, p)] = f[o:o + self.pk]
                o += self.pk
        self.ring = {}
        for io in ("in", "out"):
            for p in (0, 1):
                self.ring[(io, p)] = f[o:o + max(1, n - 1) * CTHW]
                o += max(1, n - 1) * CTHW
        self.state = {(b, j): np.zeros(d) for b in range(b0, b1) for j in range(n)}
        self.calls = 0
        self.workspace = self.ws

    def stage_io(self, parity):
        base = self.ws.data_ptr()
        nb = 8 * self.pk if self.K > 1 else 0
        rb = 8 * max(0, self.n - 1) * self.CTHW
        return _IO({"act_in": self.act[("in", parity)].data_ptr() if nb else 0,
                    "act_out": self.act[("out", parity)].data_ptr() if nb else 0, "act_bytes": nb,
                    "ring_in": self.ring[("in", parity)].data_ptr(), "ring_out": self.ring[("out", parity)].data_ptr(),
                    "ring_bytes": rb})

    def denoise_chunk(self, chunk, out):
        n, L, d, C = self.n, self.L, self.d, self.CTHW
        c = self.calls
        na, ents, oc = self.ctl.call()
        par = c & 1
        first, last = self.rank == 0, self.rank == self.K - 1
        if first:
            x = np.zeros((n, L, d)); sig = np.zeros(n); sign = np.zeros(n); lat = np.zeros((n, C))
            ring_in = self.ring[("out", (c + 1) & 1)] if self.K == 1 else self.ring[("in", par)]
            for e in ents:
                if not e["active"]:
                    continue
                j, X = e["j"], e["X"]
                sig[j] = 1.0 / (1 + X + j); sign[j] = 1.0 / (2 + X + j)
                lat[j] = chunk(X) if j == 0 else ring_in.numpy()[(j - 1) * C:j * C]
                x[j] = np.outer(np.arange(1, L + 1), np.resize(lat[j], d)) * 0.1 + sig[j]
        else:
            pkt = self.act[("in", par)].numpy()
            x = pkt[:n * L * d].reshape(n, L, d).copy()
            sig = pkt[n * L * d:n * L * d + n].copy(); sign = pkt[n * L * d + n:n * L * d + 2 * n].copy()
            lat = pkt[n * L * d + 2 * n:].reshape(n, C).copy()
        for b in range(self.b0, self.b1):
            for e in ents:
                if not e["active"]:
                    continue
                j = e["j"]
                st = self.state[(b, j)]
                st[:] = 0.5 * st + x[j].mean(0) + 0.01 * e["X"]
                x[j] = np.tanh(x[j] * (1.0 + 0.1 * b) + st)
        if not last:
            pkt = self.act[("out", par)].numpy()
            pkt[:n * L * d] = x.reshape(-1); pkt[n * L * d:n * L * d + n] = sig
            pkt[n * L * d + n:n * L * d + 2 * n] = sign; pkt[n * L * d + 2 * n:] = lat.reshape(-1)
        else:
            rout = self.ring[("out", par)].numpy()
            for e in ents:
                if not e["active"]:
                    continue
                j = e["j"]
                x0 = lat[j] - sig[j] * np.resize(x[j].mean(0), C)
                if j == n - 1:
                    out[e["X"]] = x0.copy()
                else:
                    rout[j * C:(j + 1) * C] = (1 - sign[j]) * x0 + sign[j] * 0.3
        self.calls += 1
        return oc
