// tma.cuh — Tensor Memory Accelerator (cp.async.bulk.tensor) helpers for the row-strided
// [tokens, heads, d] layout of Q/K/V.
//
// A residue class of a dilated window (tokens c, c + r, c + 2r, ...) is one TMA tensor-map
// traversal: a rank-3 map {d, heads, tokens} with element stride r on the token dimension
// loads `box_rows` class rows of one head into shared memory, 128B- (d = 64) or 64B-swizzled
// (d = 32) exactly as tc::swz lays them out.  Out-of-range coordinates (negative, or past the
// buffer) are zero-filled by the hardware.
#pragma once
#include <cuda.h> // CUtensorMap and its enums (types only: the encoder comes from cudart's entry point)
#include <stdint.h>

namespace ga {
namespace tma {

// Host: encode `map` for a row-major [ntok, H, D] tensor of 16-bit elements at `base`;
// boxes of `box_rows` token rows of one head with token stride r (box_rows * r <= 256,
// r <= 8, D * 2 in {64, 128}).  Returns false if TMA cannot express it.
bool encode_rows(CUtensorMap *map, const void *base, int64_t ntok, int H, int D, int r, int box_rows);

// Host: rank-3 map {D, H, nrows} over the token lattice base + pitch * u (u < nrows) of a
// [tokens, H, D] 16-bit tensor (token pitch `pitch` rows, any size: the lattice row stride is
// a plain global stride), boxes of `box_rows` lattice rows of one head, 128B-swizzled (D = 64).
bool encode_lattice(CUtensorMap *map, const void *base, int64_t nrows, int H, int D, int64_t pitch, int box_rows);

// Host: 2D map {H*D, ntok} of a [ntok, H, D] 16-bit tensor with a one-row {D, 1} box,
// 128B-swizzled (D = 64 only), for tile::gather4 loads of 4 arbitrary token rows of a head.
bool encode_gather(CUtensorMap *map, const void *base, int64_t ntok, int H, int D);

// Host: rank-3 map {D, H, ntok} with {D, 1, box_rows} boxes of consecutive token rows of one
// head, 128B-swizzled (D = 64): the same shared layout as box_rows / 4 gather4 loads (cached).
bool encode_block(CUtensorMap *map, const void *base, int64_t ntok, int H, int D, int box_rows);

// 4 rows (tokens y0..y3, elements [x, x + D)) -> 4 consecutive 128-byte rows of shared memory
__device__ __forceinline__ void gather4(uint32_t smem, const CUtensorMap *map, int x, int y0, int y1, int y2, int y3,
                                        uint32_t mbar)
{
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, "
                 "{%2, %3, %4, %5, %6}], [%7];" ::"r"(smem),
                 "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y0), "r"(y1), "r"(y2), "r"(y3), "r"(mbar)
                 : "memory");
}

__device__ __forceinline__ void expect_tx(uint32_t mbar, uint32_t bytes)
{
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}\n" ::"r"(mbar),
                 "r"(bytes)
                 : "memory");
}

// box at coordinates (c0 = element in d, c1 = head, c2 = token) -> shared memory, completing
// its bytes on `mbar`
__device__ __forceinline__ void load_3d(uint32_t smem, const CUtensorMap *map, int c0, int c1, int c2, uint32_t mbar)
{
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                     smem),
                 "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(mbar)
                 : "memory");
}

// shared memory -> box at coordinates (c0, c1, c2) (bulk-group completion); coordinates outside
// the tensor are not written
__device__ __forceinline__ void store_3d(const CUtensorMap *map, int c0, int c1, int c2, uint32_t smem)
{
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(smem)
                 : "memory");
}

__device__ __forceinline__ void store_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

// the bulk stores committed so far have finished reading shared memory
__device__ __forceinline__ void store_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

// every bulk store committed so far has completed (global writes done)
__device__ __forceinline__ void store_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

} // namespace tma
} // namespace ga
