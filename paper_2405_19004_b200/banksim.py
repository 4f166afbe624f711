"""Shared-memory bank model and on-chip roofline.

Python counterpart of the reference's declared-but-unimplemented
`pmg::banksim` (/root/reference/proj/include/pmg/banksim.hpp:112-139):

* `count_conflicts` — wavefronts of shared-memory requests: the maximum over
  banks of the number of distinct words routed to the bank (identical
  addresses broadcast), served per half-warp for 8-byte words
  (banksim.hpp:17-27, :112-118). ncu measures the same quantity
  (`l1tex__data_pipe_lsu_wavefronts_mem_shared`); tools/bank_search*.py use
  this model to pick the kernels' layouts.
* `shared_traffic_model` — per-patch flops and shared-memory words of one
  smoothing step following the reference's contraction sequence
  (fastdiag.cpp:164-233): per contraction, reads = |input| + n_out * n_in
  (the 1D matrix), writes = |output|; the eigenvalue scaling reads and
  writes the interior tensor once (banksim.hpp:120-133).
* `onchip_bandwidth_tbps`, `onchip_roofline` — B = SMs x banks x bank width x
  clock (binary TB/s, 17.145 for the paper's A100) and the
  bound B F / (d_r + d_w) (banksim.hpp:135-139).
"""

from __future__ import annotations

from collections import defaultdict
from dataclasses import dataclass


@dataclass(frozen=True)
class BankConfig:
    banks: int = 32
    bank_width_bytes: int = 4
    word_bytes: int = 8
    warp_size: int = 32

    def words_per_bank_group(self) -> int:
        return max(1, self.word_bytes // self.bank_width_bytes)

    def effective_banks(self) -> int:
        return self.banks // self.words_per_bank_group()

    def group_size(self) -> int:
        return self.warp_size // self.words_per_bank_group()


@dataclass
class ConflictReport:
    per_instruction: list
    total_wavefronts: int
    total_excess: int


def instruction_wavefronts(accesses, config: BankConfig = BankConfig()) -> tuple[int, int]:
    """accesses: iterable of (lane, word address) of one warp-wide request.
    Returns (wavefronts, excess over the conflict-free count)."""
    groups = defaultdict(list)
    for lane, addr in accesses:
        groups[lane // config.group_size()].append(addr)
    total = ideal = 0
    for addrs in groups.values():
        per_bank = defaultdict(set)
        for a in addrs:
            per_bank[a % config.effective_banks()].add(a)
        total += max(len(s) for s in per_bank.values())
        ideal += 1
    return total, total - ideal


def count_conflicts(instructions, config: BankConfig = BankConfig()) -> ConflictReport:
    """instructions: iterable of warp requests, each an iterable of (lane, word address)."""
    per, tw, te = [], 0, 0
    for ins in instructions:
        w, e = instruction_wavefronts(ins, config)
        per.append((w, e))
        tw += w
        te += e
    return ConflictReport(per, tw, te)


@dataclass
class TrafficCounts:
    flops: float = 0.0
    bytes_read: float = 0.0
    bytes_written: float = 0.0


def _contract(ext, n_out, direction, counts: TrafficCounts, word: int):
    n_in = ext[direction]
    out = list(ext)
    out[direction] = n_out
    size_in = 1
    for e in ext:
        size_in *= e
    size_out = 1
    for e in out:
        size_out *= e
    counts.flops += 2.0 * size_out * n_in
    counts.bytes_read += word * (size_in + n_out * n_in)
    counts.bytes_written += word * size_out
    return out


def shared_traffic_model(variant: str, degree: int, dim: int, word_bytes: int) -> TrafficCounts:
    """Per-patch on-chip traffic of one smoothing step (the reference's
    contraction sequence). variant: 'fused' (residual + solve) or 'solver'
    (the local solve only, as in the global / separate variants)."""
    if dim not in (2, 3):
        raise ValueError("dim must be 2 or 3")
    if variant not in ("fused", "solver"):
        raise ValueError("variant must be 'fused' or 'solver'")
    nc, ni = 2 * degree + 1, 2 * degree - 1
    c = TrafficCounts()
    if variant == "fused":
        # apply_patch_operator (fastdiag.cpp:211-232): dir 0, then dir 1, ... with
        # extents shrinking nc -> ni per contracted direction
        # (the "+=" contractions accumulate inside their multiply-adds)
        if dim == 2:
            for _ in range(2):  # A1 (M0 u), M1 (A0 u)
                e = _contract([nc, nc], ni, 0, c, word_bytes)
                _contract(e, ni, 1, c, word_bytes)
        else:
            e0 = _contract([nc, nc, nc], ni, 0, c, word_bytes)      # z = M0 u
            e1 = _contract(e0, ni, 1, c, word_bytes)                # t = M1 z
            _contract(e1, ni, 2, c, word_bytes)                     # r = A2 t
            _contract(e0, ni, 1, c, word_bytes)                     # t = A1 z
            _contract(e1, ni, 2, c, word_bytes)                     # r += M2 t
            e0 = _contract([nc, nc, nc], ni, 0, c, word_bytes)      # z = A0 u
            _contract(e0, ni, 1, c, word_bytes)                     # t2 = M1 z
            _contract(e1, ni, 2, c, word_bytes)                     # r += M2 t2
        c.flops += ni ** dim  # r = b - A u
    # apply_patch_inverse (fastdiag.cpp:164-192): d x S^T, scale, d x S
    e = [ni] * dim
    for d in range(dim):
        e = _contract(e, ni, d, c, word_bytes)
    c.flops += ni ** dim
    c.bytes_read += word_bytes * ni ** dim
    c.bytes_written += word_bytes * ni ** dim
    for d in range(dim):
        e = _contract(e, ni, d, c, word_bytes)
    if variant == "fused":
        c.flops += ni ** dim  # x^I += v
    return c


@dataclass(frozen=True)
class HardwareParams:
    sms: int = 148
    banks: int = 32
    bank_width_bytes: int = 4
    clock_ghz: float = 1.965


A100 = HardwareParams(sms=108, banks=32, bank_width_bytes=4, clock_ghz=1.27)
B200 = HardwareParams()


def onchip_bandwidth_tbps(hw: HardwareParams = B200) -> float:
    """B = SMs x banks x bank width x clock in the paper's "binary" TB/s
    (bytes/s / 1.024e12: 17.145 for the A100 parameter set)."""
    return hw.sms * hw.banks * hw.bank_width_bytes * hw.clock_ghz * 1e9 / 1.024e12


def onchip_roofline(flops: float, bytes_read: float, bytes_written: float, hw: HardwareParams = B200) -> float:
    """B F / (d_r + d_w) in Tflop/s (B in binary TB/s, as the paper)."""
    return onchip_bandwidth_tbps(hw) * flops / (bytes_read + bytes_written)
