"""Send/Recv transports for the oracle's partitioned runs (test infrastructure only).

PAPER.md:780-782: "The local executors communicate only via Send and Recv operations." A
message is (value or is_dead) keyed by (source, destination, channel, iteration tag); the
is_dead signal is transmitted like a value.

* ``Mailbox`` -- one in-process rendezvous table shared by the partitions, each run by its own
  thread (``Mailbox.port(rank)`` is that partition's transport).
* ``DistTransport`` -- the same over ``torch.distributed`` point-to-point (gloo on CPU): one
  float64 message per (channel, tag) = [is_dead] + flattened value, matched by a tag derived
  from (channel, tag).
"""
from __future__ import annotations

import threading
import zlib

import numpy as np


class Mailbox:
    def __init__(self):
        self._box = {}
        self._cv = threading.Condition()

    def port(self, rank: int) -> "_Port":
        return _Port(self, rank)


class _Port:
    def __init__(self, mb: Mailbox, rank: int):
        self.mb, self.rank = mb, rank

    def send(self, peer, channel, key, value, dead, shape):
        with self.mb._cv:
            k = (self.rank, peer, channel, key)
            if k in self.mb._box:
                raise RuntimeError(f"message {k} sent twice")
            self.mb._box[k] = (value, dead)
            self.mb._cv.notify_all()

    def recv(self, peer, channel, key, shape, timeout=120.0):
        k = (peer, self.rank, channel, key)
        with self.mb._cv:
            if not self.mb._cv.wait_for(lambda: k in self.mb._box, timeout=timeout):
                raise RuntimeError(f"recv {k}: no message (deadlock)")
            return self.mb._box.pop(k)


def _tag(channel, key) -> int:
    return zlib.crc32(repr((int(channel), tuple(int(k) for k in key))).encode()) & 0x3FFFFFFF


class DistTransport:
    def __init__(self):
        import torch.distributed as dist
        self.dist = dist
        self.rank = dist.get_rank()
        self.pending = []

    def send(self, peer, channel, key, value, dead, shape):
        import torch
        n = int(np.prod(shape)) if len(shape) else 1
        v = np.zeros(n) if dead else np.asarray(value, dtype=np.float64).ravel()
        msg = torch.from_numpy(np.concatenate([[1.0 if dead else 0.0], v]))
        self.pending.append((self.dist.isend(msg, dst=peer, tag=_tag(channel, key)), msg))

    def recv(self, peer, channel, key, shape):
        import torch
        n = int(np.prod(shape)) if len(shape) else 1
        buf = torch.zeros(1 + n, dtype=torch.float64)
        self.dist.recv(buf, src=peer, tag=_tag(channel, key))
        if buf[0].item() != 0.0:
            return None, True
        return buf[1:].numpy().reshape(shape).copy(), False

    def finish(self):
        for w, _ in self.pending:
            w.wait()
        self.pending.clear()
