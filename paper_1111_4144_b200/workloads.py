"""Seeded synthetic inputs shaped like BASELINE.json's configs (shared by tests, bench and
smoke).  This module holds NONE of the method's arithmetic: it only draws random matrices
and lays them out in memory.  Both the CUDA path and the oracle consume the same bits.

Recipe (BASELINE.json "configs"):
  cfg1  N=4   c64   1024   Cholesky  SoA   A = B B^H / 4  + 0.1 I
  cfg2  N=8   c64   2^20   Cholesky  SoA   A = B B^H / 8  + 0.1 I   ("interleaved")
  cfg3  N=16  c64   2^22   Cholesky  SoA   A = B B^H / 16 + 0.01 I  (reading R15)
  cfg4  N=64  c128  2^18   Cholesky  AoS   A = Q diag(lam) Q^H, Q from QR of CN(0,1),
                                           lam = 10^(3U), U ~ U[0,1) (log-uniform [1,1e3])
  cfg5  N=32  c64   2^20   LDL       AoS   A = B B^H / 32 + 0.05 I
B has i.i.d. CN(0,1) entries (re, im each N(0, 1/2): torch complex randn).  A is made
exactly Hermitian as (A + A^H)/2 with Im a_ii = 0.  Matrices are drawn in chunks of
CHUNK; chunk c of config k uses its own generator seeded from (seed, k, c), so any slice
[start, start+count) of the global batch -- e.g. one rank's shard -- is generated
independently and bit-identically to the same slice of an unsharded run (same device type).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Tuple

import torch

CHUNK = 4096


@dataclass(frozen=True)
class Config:
    cid: int
    n: int
    dtype: torch.dtype
    batch: int
    method: str            # "chol" | "ldl"
    layout: str            # "soa" | "aos"
    kind: str              # "bbh" | "spectral"
    divisor: float = 1.0   # A = B B^H / divisor + delta I
    delta: float = 0.0
    desc: str = ""
    task: str = "inv"      # "inv" (the hot path) | "solve" (§8(f) f1: A x = y) | "nonherm" (f2) | "fxp" (f4)
    qm: int = 2            # fixed-point format Q(qm, qf) of the f4 study
    qf: int = 13

    @property
    def elem_bytes(self) -> int:
        return 8 if self.dtype == torch.complex64 else 16


CONFIGS = {
    1: Config(1, 4, torch.complex64, 1024, "chol", "soa", "bbh", 4.0, 0.1,
              "1024 c64 HPD 4x4, A = BB^H/4 + 0.1I, Cholesky + proposed, seed 0"),
    2: Config(2, 8, torch.complex64, 1 << 20, "chol", "soa", "bbh", 8.0, 0.1,
              "2^20 c64 HPD 8x8, A = BB^H/8 + 0.1I, interleaved (SoA) batch layout"),
    3: Config(3, 16, torch.complex64, 1 << 22, "chol", "soa", "bbh", 16.0, 0.01,
              "2^22 c64 HPD 16x16, A = BB^H/16 + 0.01I, interleaved (SoA)"),
    4: Config(4, 64, torch.complex128, 1 << 18, "chol", "aos", "spectral", 1.0, 0.0,
              "2^18 c128 HPD 64x64, A = Q diag(lam) Q^H, lam log-uniform [1,1e3], one matrix per CTA"),
    5: Config(5, 32, torch.complex64, 1 << 20, "ldl", "aos", "bbh", 32.0, 0.05,
              "2^20 c64 HPD 32x32, A = BB^H/32 + 0.05I, LDL R*DR + proposed"),
    # SURVEY §8(f) f1 (next row, not a BASELINE.json config): the cfg2 matrices, one
    # right-hand side y ~ CN(0, I) each, solved by eqs. (5)-(7)
    6: Config(6, 8, torch.complex64, 1 << 20, "chol", "soa", "bbh", 8.0, 0.1,
              "2^20 c64 HPD 8x8 systems A x = y (cfg2 matrices, y ~ CN(0,I)), Cholesky solve eqs. 5-7, "
              "interleaved", task="solve"),
    # SURVEY §8(f) f1 at the lane-group sizes: the cfg3 matrices (n = 16) with one right-hand
    # side each, solved by eqs. 5-7 (k_grp_solve)
    9: Config(9, 16, torch.complex64, 1 << 22, "chol", "soa", "bbh", 16.0, 0.01,
              "2^22 c64 HPD 16x16 systems A x = y (cfg3 matrices, y ~ CN(0,I)), Cholesky solve eqs. 5-7, "
              "interleaved", task="solve"),
    # SURVEY §8(f) f2 (next row): non-Hermitian D = I + B / (2 sqrt(n)), B i.i.d. CN(0,1) (a
    # channel-like matrix near the identity; the paper gives no workload), D^-1 = D* (DD*)^-1
    7: Config(7, 8, torch.complex64, 1 << 20, "chol", "soa", "nonherm", 2.0 * 8 ** 0.5, 1.0,
              "2^20 c64 non-Hermitian 8x8 D = I + B/(2 sqrt 8), D^-1 = D*(DD*)^-1 (P:135-141), interleaved",
              task="nonherm"),
    # SURVEY §8(f) f4 (next row): the fixed-point accuracy study of §IV.C with 16-bit words
    # Q4.11 (reading F8: SPEC's Q2.13 saturates X = A^-1 in ~80 % of trials, |x| ~ 1/0.1),
    # n = 16, SPEC.md's ensemble: G re/im ~ U[-1, 1], A = G G^H / n + 0.1 I, scaled
    # so max |a_ij| <= 0.9 * (2^m - 2^-f), then quantized (round half to even, saturated)
    8: Config(8, 16, torch.complex128, 1 << 16, "chol", "aos", "fxp", 16.0, 0.1,
              "2^16 Q4.11 fixed-point HPD 16x16 (SPEC ensemble), Cholesky + proposed inversion emulated "
              "in integer arithmetic (F1-F7)", task="fxp", qm=4, qf=11),
}


def chunk_seed(seed: int, cid: int, chunk: int) -> int:
    # splitmix64-style mixing of (seed, config, chunk) into a 63-bit torch seed
    x = (seed * 0x9E3779B97F4A7C15 + cid * 0xBF58476D1CE4E5B9 + chunk * 0x94D049BB133111EB) & (2**64 - 1)
    x ^= x >> 31
    x = (x * 0xD6E8EB7A8B3F7C5B) & (2**64 - 1)
    x ^= x >> 29
    return x & (2**63 - 1)


def _hermitise(A: torch.Tensor) -> torch.Tensor:
    A = (A + A.conj().transpose(-1, -2)) * 0.5
    d = torch.diagonal(A, dim1=-2, dim2=-1)
    d.imag.zero_()
    return A


def _gen_chunk(cfg: Config, chunk: int, count: int, device, seed: int) -> torch.Tensor:
    g = torch.Generator(device=device)
    g.manual_seed(chunk_seed(seed, cfg.cid, chunk))
    n = cfg.n
    if cfg.kind == "bbh":
        B = torch.randn(count, n, n, dtype=cfg.dtype, device=device, generator=g)
        A = torch.matmul(B, B.conj().transpose(-1, -2)) / cfg.divisor
        A = A + cfg.delta * torch.eye(n, dtype=cfg.dtype, device=device)
        return _hermitise(A)
    if cfg.kind == "nonherm":            # D = delta I + B / divisor (not Hermitian)
        B = torch.randn(count, n, n, dtype=cfg.dtype, device=device, generator=g)
        return B / cfg.divisor + cfg.delta * torch.eye(n, dtype=cfg.dtype, device=device)
    # spectral: A = Q diag(lam) Q^H
    G = torch.randn(count, n, n, dtype=cfg.dtype, device=device, generator=g)
    U = torch.rand(count, n, dtype=torch.float64, device=device, generator=g)
    lam = torch.pow(10.0, 3.0 * U).to(cfg.dtype)
    Q, _ = torch.linalg.qr(G)
    A = torch.matmul(Q * lam[:, None, :], Q.conj().transpose(-1, -2))
    return _hermitise(A)


def generate(cfg: Config, start: int = 0, count: Optional[int] = None, device="cpu",
             seed: int = 0) -> torch.Tensor:
    """Matrices [start, start+count) of config `cfg`'s global batch as a contiguous (AoS)
    (count, n, n) tensor on `device`."""
    if count is None:
        count = cfg.batch - start
    out = torch.empty(count, cfg.n, cfg.n, dtype=cfg.dtype, device=device)
    pos = start
    while pos < start + count:
        c = pos // CHUNK
        c0 = c * CHUNK
        take = min(c0 + CHUNK, start + count) - pos
        chunk = _gen_chunk(cfg, c, CHUNK, device, seed)
        out[pos - start:pos - start + take] = chunk[pos - c0:pos - c0 + take]
        pos += take
    return out


def generate_rhs(cfg: Config, start: int = 0, count: Optional[int] = None, device="cpu",
                 seed: int = 0) -> torch.Tensor:
    """Right-hand sides [start, start+count) for config `cfg` (f1 solve): (count, n), entries
    i.i.d. CN(0,1); chunk-keyed like `generate` (stream id 1000 + config id)."""
    if count is None:
        count = cfg.batch - start
    out = torch.empty(count, cfg.n, dtype=cfg.dtype, device=device)
    pos = start
    while pos < start + count:
        c = pos // CHUNK
        c0 = c * CHUNK
        take = min(c0 + CHUNK, start + count) - pos
        g = torch.Generator(device=device)
        g.manual_seed(chunk_seed(seed, 1000 + cfg.cid, c))
        chunk = torch.randn(CHUNK, cfg.n, dtype=cfg.dtype, device=device, generator=g)
        out[pos - start:pos - start + take] = chunk[pos - c0:pos - c0 + take]
        pos += take
    return out


def vec_layout(Y: torch.Tensor, layout: str, ld: Optional[int] = None) -> Tuple[torch.Tensor, torch.Tensor]:
    """Copy contiguous (batch, n) vectors into `layout` ("aos": contiguous; "soa": element i of
    system b at planes[i, b], ld >= batch).  Returns (storage, (batch, n) view)."""
    batch, n = Y.shape
    if layout == "aos":
        buf = Y.contiguous()
        return buf, buf
    ld = batch if ld is None else ld
    planes = torch.empty(n, ld, dtype=Y.dtype, device=Y.device)
    planes[:, :batch] = Y.t()
    if ld > batch:
        planes[:, batch:] = float("nan")
    return planes, torch.as_strided(planes, (batch, n), (1, ld))


def quantize(x: torch.Tensor, m: int, f: int) -> torch.Tensor:
    """Real tensor -> int64 raws of Q(m, f): round half to even of x 2^f (torch.round), saturated
    to [-2^(m+f), 2^(m+f) - 1] (SPEC.md quantize; DESIGN reading F1-F2)."""
    r = torch.round(x.to(torch.float64) * float(2 ** f))
    return r.clamp(-float(2 ** (m + f)), float(2 ** (m + f) - 1)).to(torch.int64)


def generate_fxp(cfg: Config, start: int = 0, count: Optional[int] = None, device="cpu",
                 seed: int = 0) -> Tuple[torch.Tensor, torch.Tensor]:
    """f4 study inputs: (A complex128 (count, n, n) -- the unquantized matrices the double
    reference inverts -- and A_raw int64 (count, n, n, 2), its Q(qm, qf) quantization).
    Chunk-keyed like `generate`."""
    if count is None:
        count = cfg.batch - start
    n = cfg.n
    out = torch.empty(count, n, n, dtype=torch.complex128, device=device)
    rho = 0.9 * (2.0 ** cfg.qm - 2.0 ** -cfg.qf)
    pos = start
    while pos < start + count:
        c = pos // CHUNK
        c0 = c * CHUNK
        take = min(c0 + CHUNK, start + count) - pos
        g = torch.Generator(device=device)
        g.manual_seed(chunk_seed(seed, cfg.cid, c))
        U = torch.rand(CHUNK, n, n, 2, dtype=torch.float64, device=device, generator=g) * 2.0 - 1.0
        G = torch.complex(U[..., 0], U[..., 1])
        A = torch.matmul(G, G.conj().transpose(-1, -2)) / cfg.divisor
        A = A + cfg.delta * torch.eye(n, dtype=torch.complex128, device=device)
        A = _hermitise(A)
        mx = A.abs().amax(dim=(1, 2))
        A = A / torch.clamp(mx / rho, min=1.0)[:, None, None]
        out[pos - start:pos - start + take] = A[pos - c0:pos - c0 + take]
        pos += take
    raw = torch.stack([quantize(out.real, cfg.qm, cfg.qf), quantize(out.imag, cfg.qm, cfg.qf)], dim=-1)
    return out, raw.contiguous()


def soa_view(planes: torch.Tensor, batch: int, n: int) -> torch.Tensor:
    """(batch, n, n) view of an interleaved buffer `planes` of shape (n*n, ld), ld >= batch:
    element (i, j) of matrix b at planes[i*n + j, b]."""
    ld = planes.shape[1]
    return torch.as_strided(planes, (batch, n, n), (1, n * ld, ld))


def to_layout(A: torch.Tensor, layout: str, ld: Optional[int] = None) -> Tuple[torch.Tensor, torch.Tensor]:
    """Copy contiguous (batch, n, n) matrices into `layout`.  Returns (storage, view)."""
    batch, n = A.shape[0], A.shape[1]
    if layout == "aos":
        buf = A.contiguous()
        return buf, buf
    ld = batch if ld is None else ld
    planes = torch.empty(n * n, ld, dtype=A.dtype, device=A.device)
    planes[:, :batch] = A.reshape(batch, n * n).t()
    if ld > batch:
        planes[:, batch:] = float("nan")
    return planes, soa_view(planes, batch, n)


def empty_like_layout(view: torch.Tensor) -> torch.Tensor:
    """Output tensor with the same (batch, n, n) strides as `view`."""
    return torch.empty_strided(view.shape, view.stride(), dtype=view.dtype, device=view.device)


def shard(rank: int, world: int, batch: int) -> Tuple[int, int]:
    """Contiguous slice [start, start+count) of `batch` owned by `rank` of `world`."""
    base, rem = divmod(batch, world)
    start = rank * base + min(rank, rem)
    return start, base + (1 if rank < rem else 0)
