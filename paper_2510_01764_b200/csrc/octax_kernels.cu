// octax_kernels.cu -- sm_100a kernels of the batched Octax environment step.
//
// One thread = one environment (CHIP-8 VM), 128 envs per CTA.  Per step:
//   * the 4 KB pristine image (font + ROM) is staged once per CTA into shared
//     memory with a TMA bulk copy (cp.async.bulk + mbarrier);
//   * the CTA's 32 KB block of the newest display slot of the HBM ring is staged
//     into the shared-memory framebuffer with one more TMA bulk copy (32 x u64
//     rows per env, XOR-swizzled: bank-conflict free both for "one row of 32 envs"
//     and "32 rows of one env"; the ring keeps the same swizzle); obs planes 0..2
//     are written in row order with 16-B lane chunks, planes 0,1 streamed from
//     the ring one env per VM cycle behind the interpreter;
//   * fetch + decode is one L1 load of the word predecoded per handle at every PC
//     (flags, skip truth table, stack delta, register offsets, NNN; make_entry in
//     octax_dev.cuh), issued one VM cycle ahead; a PC in a dirty RAM block decodes
//     on the device in a vote-gated slow path;
//   * the interpreter loop (frame_skip x instructions_per_frame cycles,
//     P:142-146) is WARP-UNIFORM: every lane runs the same straight-line,
//     predicated core for the cheap opcode classes (no divergent dispatch
//     tree), and the rare / heavy classes (DXYN, CXNN, 00E0, FX33/55/65) are
//     vote-gated blocks executed once per warp when any lane needs them;
//   * DXYN, chosen per warp and cycle from the drawing lanes' row
//     counts: grouped (each drawer's rows spread over a group of lanes, one row
//     step for up to 32 / maxr drawers, collisions from one ballot), single-row,
//     lane-parallel (each lane its own rows), or cooperative (prefix-summed rows
//     of all drawers over the 32 lanes);
//   * score / termination bytecode -> reward, done; same-step
//     auto-reset with startup segments (A10), also warp-uniform;
//   * the epilogue bulk-stores the framebuffer block as the new ring slot and
//     writes obs plane 3;
//   * per-CTA integer episode statistics -> 4 int64 atomics per CTA.
// Semantics follow DESIGN.md readings A1..A32; nothing here is shared with
// the CPU oracle in oracle/.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cassert>
#include <cstdint>

#include "octax_dev.cuh"

// Checked build (liboctax_checked.so, -DOCTAX_CHECKS): device-side bounds asserts on
// every computed shared / global index -- the substitute for compute-sanitizer, which
// is closed on this GPU pool.
#ifdef OCTAX_CHECKS
#define OCTAX_CHECK(c) assert(c)
#else
#define OCTAX_CHECK(c) ((void)0)
#endif

namespace octax {

constexpr unsigned kFull = 0xffffffffu;

// Programmatic dependent launch (OCTAX_PDL): step / rollout kernels are launched with programmatic
// stream serialization, so the next launch's CTAs are scheduled while this grid drains; each
// waits (griddepcontrol.wait) for the preceding grid to complete and its writes to be visible
// before touching any state, so stream order is kept exactly, only the launch gap overlaps.
#ifndef OCTAX_PDL  // A/B knob: 0 = plain launches and no griddepcontrol instructions
#define OCTAX_PDL 1
#endif
__device__ __forceinline__ void pdl_enter() {
#if OCTAX_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
#ifndef OCTAX_LANE_DRAW_MAX
#define OCTAX_LANE_DRAW_MAX 8
#endif
#ifndef OCTAX_GROUP_MIN_ROWS
#define OCTAX_GROUP_MIN_ROWS 3
#endif
constexpr uint32_t kLaneDrawMax = OCTAX_LANE_DRAW_MAX;  // rows: lane-parallel DXYN up to this, cooperative above
constexpr uint32_t kGroupMinRows = OCTAX_GROUP_MIN_ROWS;  // grouped DXYN from this many rows (A/B knobs)
static_assert(kLaneDrawMax <= 8u, "the lane-parallel fast path realigns an 8-byte sprite window");
// ceil(2^32 / m): lane / m = umulhi(lane, kRecip[m]) exactly for lane < 2^16 (m = 2..15)
__constant__ uint32_t kRecip[16] = {0u, 0u, 0x80000000u, 0x55555556u, 0x40000000u, 0x33333334u,
                                    0x2AAAAAABu, 0x24924925u, 0x20000000u, 0x1C71C71Du, 0x1999999Au,
                                    0x1745D175u, 0x15555556u, 0x13B13B14u, 0x12492493u, 0x11111112u};

// framebuffer / ring row swizzle: row r of env e sits at position r ^ (e & kSwz).  14 keeps row
// pairs (2k, 2k+1) in order inside every 16-B chunk, so obs rows move as 16-B stores; 8 envs
// (not 16) then differ in the position of a given row (A/B: +0.1..0.6% over 15).
#ifndef OCTAX_SWZ
#define OCTAX_SWZ 14
#endif
constexpr uint32_t kSwz = OCTAX_SWZ;

struct __align__(128) Smem {
  uint8_t img[kImageBytes];                  // pristine image (TMA destination) ...
  uint32_t dtab[kDescEntries];               // ... immediately followed by the decode table
  uint64_t fb[kBlock * 32];                  // framebuffer rows, bit 63-x = pixel x, swizzled
  uint8_t V[16 * kBlock];                    // V[k] of env t: its own bank (see vbase / VREG)
  uint16_t stk[16 * kBlock];                 // stk[k*kBlock + tid]
  uint32_t dprm[kBlock / 32][32];            // DXYN owner params (x0 | y0 << 6 | base << 11)
  uint8_t down[kBlock / 32][32];             // DXYN item -> owner lane map
  unsigned long long red[4][kBlock / 32];    // per-warp statistics
  unsigned long long bar;                    // mbarrier for the image copy
};

size_t smem_bytes() { return sizeof(Smem); }

// byte `a` of the CTA's shared-memory copy of the pristine image (zeros, font, ROM)
#define IMG(a) ((uint32_t)sm.img[a])

// framebuffer row `r` of CTA-local env `e`: XOR swizzle on the low 4 row bits
__device__ __forceinline__ uint32_t fb_idx(uint32_t e, uint32_t r) {
  OCTAX_CHECK(e < (uint32_t)kBlock && r < 32u);
  return e * 32u + (r ^ (e & kSwz));
}

__device__ __forceinline__ uint64_t bswap64(uint64_t v) {
  uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
  return ((uint64_t)__byte_perm(lo, 0, 0x0123) << 32) | (uint64_t)__byte_perm(hi, 0, 0x0123);
}

// Philox4x32-10, first output word (Random123 algorithm; reading A12).
__device__ __forceinline__ uint32_t philox_out0(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  return c0;
}

// ---------------------------------------------------------------- TMA bulk copies
// One elected thread stages the 5 KB image (+ decode table) and, in a step, the CTA's
// 32 KB framebuffer block of ring slot `h` into shared memory on one mbarrier.
__device__ __forceinline__ void stage_issue(Smem &sm, const uint8_t *img, const uint64_t *fb_src) {
  uint32_t bar = (uint32_t)__cvta_generic_to_shared(&sm.bar);
  const uint32_t bytes = kStageBytes + (fb_src ? (uint32_t)sizeof(sm.fb) : 0u);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
  const uint32_t dst = (uint32_t)__cvta_generic_to_shared(sm.img);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(img), "r"(kStageBytes), "r"(bar)
      : "memory");
  if (fb_src) {
    const uint32_t fdst = (uint32_t)__cvta_generic_to_shared(sm.fb);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(fdst),
        "l"(fb_src), "r"((uint32_t)sizeof(sm.fb)), "r"(bar)
        : "memory");
  }
}

__device__ __forceinline__ void stage_wait(Smem &sm) {
  uint32_t bar = (uint32_t)__cvta_generic_to_shared(&sm.bar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(bar)
        : "memory");
  }
}

// CTA framebuffer block -> one ring slot (bulk store; caller fenced + synced the CTA)
__device__ __forceinline__ void fb_store_issue(const Smem &sm, uint64_t *dst) {
  const uint32_t src = (uint32_t)__cvta_generic_to_shared(sm.fb);
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src),
               "r"((uint32_t)sizeof(sm.fb))
               : "memory");
}

// ring slot `slot` of handle-local env `e` (32 positions; position j holds row j ^ (e & kSwz))
__device__ __forceinline__ uint64_t *ring_at(const StepParams &p, uint32_t slot, uint64_t e) {
  OCTAX_CHECK(slot < 4u && e * 32u < p.s.ring_stride);
  return p.s.ring + (uint64_t)slot * p.s.ring_stride + e * 32u;
}

// obs plane `pl` of an env from one lane's 16-B chunk of positions 2l, 2l+1 = rows ra, ra^1
// with ra = 2l ^ (e & kSwz); with the even swizzle ra is even, so the chunk is one 16-B store.
__device__ __forceinline__ void put_rows(uint64_t *ob_env, uint32_t pl, uint32_t ra, uint4 q) {
  if ((kSwz & 1u) == 0u) {  // even swizzle: ra is even, the chunk is rows ra, ra+1 in order
    __stcs(reinterpret_cast<uint4 *>(ob_env + pl * 32u + ra), q);
  } else {
    __stcs(ob_env + pl * 32u + ra, ((uint64_t)q.y << 32) | q.x);
    __stcs(ob_env + pl * 32u + (ra ^ 1u), ((uint64_t)q.w << 32) | q.z);
  }
}

// Obs rows 2k, 2k+1 of env el from the shared framebuffer as ONE 16-B streaming store, for the
// two-envs-per-pass loops (lanes 0-15 env el even, 16-31 env el odd: hh = el & 1).  Lane chunk
// l2 = 2(lane & 15) covers positions l2, l2+1 = rows l2 ^ s, (l2+1) ^ s (s = el & kSwz); for an
// odd s (OCTAX_SWZ=15) that pair is reversed, so the lane reads positions l2 ^ (s & 1),
// l2 ^ (s & 1) ^ 1 instead and writes rows (l2 ^ s) & ~1 onwards in order.
__device__ __forceinline__ void put_pair(const uint64_t *fb_env, uint64_t *ob_env, uint32_t pl, uint32_t l2,
                                         uint32_t s) {
  if ((kSwz & 1u) == 0u) {  // even swizzle: positions l2, l2+1 are one 16-B chunk (one LDS.128,
                            // conflict free; two 8-B loads were 2-way conflicted)
    __stcs(reinterpret_cast<ulonglong2 *>(ob_env + pl * 32u + (l2 ^ s)),
           *reinterpret_cast<const ulonglong2 *>(fb_env + l2));
    return;
  }
  const uint32_t hh = s & 1u;
  const uint64_t lo = fb_env[l2 ^ hh], hi = fb_env[l2 ^ hh ^ 1u];
  __stcs(reinterpret_cast<ulonglong2 *>(ob_env + pl * 32u + ((l2 ^ s) & ~1u)), make_ulonglong2(lo, hi));
}

// ---------------------------------------------------------------- lane state
struct Lane {
  uint32_t pc, sp, dt, st, halted, draw, episode;
  bool run;         // inside a cycle loop: this lane participates and has not halted
  uint32_t I;       // index register; only its low 16 bits are meaningful (FX1E wraps, A18)
  uint32_t keys;    // held key mask, 16 bits replicated into both halves
  uint32_t wvm;     // descriptor bits that write VX this step: D_WVX, + D_WAIT if a key is held
  uint32_t stay;    // entry bits that keep the PC: D_WAIT if no key is held (FX0A re-executes), E_BAD
  uint32_t kidx;    // lowest held key (FX0A result)
  uint64_t dirty;   // copy-on-write mask: block b (64 B) of RAM lives in HBM
  uint8_t *ram;
  uint32_t stk_dirty;
  uint2 dec;        // predecoded word at pc, loaded one cycle ahead (latency hidden)
};

// V[k] of CTA lane tid: warp w's 32 lanes x 16 registers occupy 512 B, register k of
// lane l at word 32 * (k >> 2) + l, byte k & 3 -- every lane's registers sit in its own
// bank, so any per-lane mix of register indices is conflict free.
__device__ __forceinline__ uint32_t vbase(int tid) {
  return (((uint32_t)tid >> 5) << 9) | (((uint32_t)tid & 31u) << 2);
}
#define VREG(k) sm.V[vbase(tid) | (((uint32_t)(k) >> 2) << 7) | ((uint32_t)(k) & 3u)]

// the key mask held for a step / startup segment and the per-step FX0A constants
__device__ __forceinline__ void set_keys(Lane &L, uint32_t km) {
  L.keys = km * 0x10001u;
  L.wvm = km ? (D_WVX | D_WAIT) : D_WVX;
  L.stay = (km ? 0u : D_WAIT) | E_BAD;  // E_BAD: a faulting entry keeps its PC (cycle<Q0, false>)
  L.kidx = (uint32_t)(__ffs(km) - 1);
}
// XOR a sprite-row mask into a framebuffer row, returning the row's old value (VF = old & mask).
// (Two native 32-bit ATOMS.XOR instead measured -0.3..-0.6%; sm_100 has no native 64-bit one.)
__device__ __forceinline__ uint64_t xor_row(uint64_t *row, uint64_t m) {
  const uint64_t old = *row;
  *row = old ^ m;
  return old;
}

// Flag test written with a two-bit mask (kPad is never set in an entry): keeps the
// compiler from lowering a single-bit test to shift + and + compare (one LOP3 instead).
constexpr uint32_t kPad = 1u << 24;
#define HAS(d, F) (((d) & ((F) | kPad)) != 0u)


__device__ __forceinline__ uint32_t rd(const Smem &sm, const StepParams &p, const Lane &L, uint32_t a) {
  OCTAX_CHECK(a < 4096u);
  return ((L.dirty >> (a >> 6)) & 1ull) ? (uint32_t)L.ram[a] : IMG(a);
}

__device__ __forceinline__ void wr(const Smem &sm, const StepParams &p, Lane &L, uint32_t a, uint32_t v) {
  OCTAX_CHECK(a < 4096u);
  uint32_t b = a >> 6;
  if (!((L.dirty >> b) & 1ull)) {  // copy-on-write: materialise the 64-B block
    const uint4 *src = reinterpret_cast<const uint4 *>(sm.img + b * 64);
    uint4 *dst = reinterpret_cast<uint4 *>(L.ram + b * 64);
    dst[0] = src[0]; dst[1] = src[1]; dst[2] = src[2]; dst[3] = src[3];
    L.dirty |= 1ull << b;
  }
  L.ram[a] = (uint8_t)v;
}

__device__ __forceinline__ void power_on(Smem &sm, Lane &L, const StepParams &p, int tid) {
#pragma unroll
  for (int j = 0; j < 4; ++j) *reinterpret_cast<uint32_t *>(&sm.V[vbase(tid) | (j << 7)]) = 0u;
#pragma unroll
  for (int k = 0; k < 16; ++k) sm.stk[k * kBlock + tid] = 0;
#pragma unroll
  for (int r = 0; r < 32; ++r) sm.fb[tid * 32 + r] = 0;
  L.pc = 0x200; L.I = 0; L.sp = 0; L.dt = 0; L.st = 0; L.halted = 0; L.draw = 0;
  set_keys(L, 0u);
  L.dirty = 0;
  L.dec = __ldg(p.s.dec + 0x200);
  L.stk_dirty = 1;
}

// shared-memory stack -> the env's 32-B HBM stack row
__device__ __forceinline__ void store_stack(const Smem &sm, const StepParams &p, int tid, uint64_t env) {
  uint32_t sw[8];
#pragma unroll
  for (int k = 0; k < 8; ++k)
    sw[k] = (uint32_t)sm.stk[(2 * k) * kBlock + tid] | ((uint32_t)sm.stk[(2 * k + 1) * kBlock + tid] << 16);
  p.s.stack[env * 2] = make_uint4(sw[0], sw[1], sw[2], sw[3]);
  p.s.stack[env * 2 + 1] = make_uint4(sw[4], sw[5], sw[6], sw[7]);
}

// Cooperative DXYN for every lane with do_draw (must be called by all 32 lanes).
// Work item k of the warp = row r of owner lane j.  Row counts are prefix-summed
// with 4 ballots (counts are 4-bit), owners publish (lane, params) into a per-warp
// smem map at their start item, and each item finds its owner as the highest
// start bit at or below it (one REDUX.OR + FLO), so a pass costs no shuffle chain.
template <bool SCAT>  // SCAT: the warp's lanes hold scattered env ids (reset_kernel)
__device__ __noinline__ void draw_coop(Smem &sm, const Lane &L, const StepParams &p, int tid, int lane,
                                          uint64_t block0, bool do_draw, uint32_t x0, uint32_t y0, uint32_t base,
                                          uint32_t n, bool vfw, uint32_t quirks) {
  const bool wrap = (quirks & 8u) != 0;
  const uint32_t nrows = do_draw ? (wrap ? n : min(n, 32u - y0)) : 0u;
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t excl = 0, total = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const uint32_t B = __ballot_sync(kFull, (nrows >> b) & 1u);
    excl += (uint32_t)__popc(B & lt) << b;
    total += (uint32_t)__popc(B) << b;
  }
  const uint32_t warp = (uint32_t)tid >> 5, wl = (uint32_t)tid & ~31u;
  sm.dprm[warp][lane] = x0 | (y0 << 6) | (base << 11);
  uint32_t hitmask = 0;
  for (uint32_t b0 = 0; b0 < total; b0 += 32) {
    const bool inw = nrows != 0u && excl >= b0 && excl < b0 + 32u;
    if (inw) sm.down[warp][excl - b0] = (uint8_t)lane;
    const uint32_t M = __reduce_or_sync(kFull, inw ? 1u << (excl - b0) : 0u);
    const uint32_t cover = __ballot_sync(kFull, nrows != 0u && excl < b0 && excl + nrows > b0);
    const uint32_t cj = cover ? (uint32_t)(__ffs(cover) - 1) : 0u;
    const uint32_t cex = __shfl_sync(kFull, excl, cj);
    __syncwarp();
    const uint32_t k = b0 + (uint32_t)lane;
    const uint32_t mk = M & (0xFFFFFFFFu >> (31 - lane));
    uint32_t j, r;
    if (mk) {
      const uint32_t pos = 31u - (uint32_t)__clz(mk);
      j = sm.down[warp][pos];
      r = (uint32_t)lane - pos;
    } else {
      j = cj;
      r = k - cex;
    }
    const uint64_t dj = __shfl_sync(kFull, L.dirty, j);
    // owner's RAM backing: env block0 + wl + j, or (SCAT) the owner lane's own pointer
    const uint8_t *rj = SCAT ? reinterpret_cast<const uint8_t *>(
                                   __shfl_sync(kFull, reinterpret_cast<unsigned long long>(L.ram), j))
                             : p.s.ram + (block0 + wl + j) * 4096ull;
    bool hit = false;
    if (k < total) {
      const uint32_t pj = sm.dprm[warp][j];
      const uint32_t xj = pj & 63u, yy = (((pj >> 6) & 31u) + r) & 31u, a = (pj >> 11) + r;
      uint32_t byte = 0;
      if (a <= 0xFFFu)
        byte = ((dj >> (a >> 6)) & 1ull) ? (uint32_t)rj[a] : IMG(a);
      uint64_t m = (uint64_t)byte << 56;
      m = bswap64(wrap ? ((m >> xj) | (xj ? (m << (64u - xj)) : 0ull)) : (m >> xj));
      uint64_t *row = &sm.fb[fb_idx(wl + j, yy)];
      const uint64_t old = *row;
      *row = old ^ m;
      hit = (old & m) != 0ull;
    }
    hitmask |= __reduce_or_sync(kFull, hit ? (1u << j) : 0u);
    __syncwarp();
  }
  if (vfw) VREG(15) = (uint8_t)((hitmask >> lane) & 1u);
}

// DXYN, lane-parallel: every drawing lane XORs its own rows, loop bound = the
// warp's largest row count (uniform).  Fast variants (sprite bytes from the smem
// image, clip or wrap) are branch-free: rows past a lane's count XOR a zero mask
// into its own (lane-private) rows.  Any dirty sprite block -> general loop.
// The framebuffer holds rows in packed byte order (byte b = pixels 8b..8b+7, MSB
// leftmost), so the mask is built as bswap16(sprite << 8 >> (x0 & 7)) << 8*(x0 >> 3).
__device__ __forceinline__ void draw_lanes(Smem &sm, Lane &L, const StepParams &p, int tid, bool do_draw,
                                           uint32_t x0, uint32_t y0, uint32_t base, uint32_t nrows, uint32_t maxr,
                                           bool wdirty, uint32_t quirks, bool vfw) {
  const bool wrap = (quirks & 8u) != 0;
  bool slowb = do_draw & (base + 15u > 0xFFFu);
  if (wdirty) slowb |= do_draw & (((L.dirty >> (base >> 6)) & 3ull) != 0ull);
  const uint32_t sh = x0 & 7u, q8 = (x0 >> 3) * 8u, swz = (uint32_t)tid & kSwz;
  uint64_t *rows = &sm.fb[(uint32_t)tid * 32u];
  // lanes without rows XOR a zero mask into rows of their own env; start them at row tid & 0x11,
  // which puts the 16 lanes of each half-warp on 16 distinct bank pairs for every r < 8 (instead
  // of wherever their VY points), so only the drawing lanes can bank-conflict
  y0 = nrows != 0u ? y0 : ((uint32_t)tid & 0x11u);
  uint64_t hit = 0;
  if (!wrap && !__any_sync(kFull, slowb)) {
    // sprite bytes base..base+7 realigned from three 32-bit image words
    const uint32_t *w = reinterpret_cast<const uint32_t *>(sm.img + (base & 0xFFCu));
    const uint32_t off8 = (base & 3u) * 8u, w0 = w[0], w1 = w[1], w2 = w[2];
    const uint32_t v0 = __funnelshift_r(w0, w1, off8), v1 = __funnelshift_r(w1, w2, off8);
    const uint32_t sl = 8u - sh;
#pragma unroll
    for (uint32_t r = 0; r < kLaneDrawMax; ++r) {
      if (r >= maxr) break;
      uint32_t byte = ((r < 4 ? v0 : v1) >> (8u * (r & 3u))) & 255u;
      byte = r < nrows ? byte : 0u;
      const uint64_t m = (uint64_t)__byte_perm(byte << sl, 0, 0x4401) << q8;
      uint64_t *row = rows + (((y0 + r) & 31u) ^ swz);
      const uint64_t old = xor_row(row, m);
      hit |= old & m;
    }
  } else {
    for (uint32_t r = 0; r < maxr; ++r) {
      const uint32_t a = base + r;
      uint32_t byte = (r < nrows && a <= 0xFFFu) ? rd(sm, p, L, a) : 0u;
      const uint64_t w = (uint64_t)__byte_perm((byte << 8) >> sh, 0, 0x4401);
      const uint64_t m = wrap ? ((w << q8) | (q8 ? (w >> (64u - q8)) : 0ull)) : (w << q8);
      uint64_t *row = rows + (((y0 + r) & 31u) ^ swz);
      const uint64_t old = xor_row(row, m);
      hit |= old & m;
    }
  }
  if (vfw) VREG(15) = (uint8_t)(hit != 0ull);
}

// DXYN, grouped, one pass: the k drawing lanes of the warp (k <= 32 / G, G = 2^lg >= the
// warp's largest row count) publish packed parameters to a per-warp smem slot by rank;
// lane r of group g XORs row r of drawer g, so all drawers cost one row step.  The
// collision bits come back with one ballot.  dm = lanes with >= 1 row; DXY0 -> VF = 0.
template <bool DIRTY, bool SCAT>  // DIRTY: some lane of the warp has private RAM (sprite bytes may
                                   // live in HBM); SCAT: scattered env ids (reset_kernel)
__device__ __forceinline__ void draw_groups(Smem &sm, const Lane &L, const StepParams &p, int tid, int lane,
                                            uint64_t block0, uint32_t dm, uint32_t x0, uint32_t y0, uint32_t base,
                                            uint32_t nrows, uint32_t m, bool wdirty, uint32_t quirks, bool vfw) {
  const bool wrap = (quirks & 8u) != 0;
  const uint32_t warp = (uint32_t)tid >> 5, wl = (uint32_t)tid & ~31u;
  const bool mine = ((dm >> lane) & 1u) != 0u;
  const uint32_t rank = (uint32_t)__popc(dm & ((1u << lane) - 1u));
  // unconditional (no branch): non-drawers write slot 31, never read (<= 10 drawers here)
  sm.dprm[warp][mine ? rank : 31u] = x0 | (y0 << 6) | (base << 11) | (nrows << 23) | ((uint32_t)lane << 27);
  __syncwarp();
  // group g = lane / m, row r = lane % m (m = the warp's largest row count, 3..15)
  const uint32_t g = __umulhi((uint32_t)lane, kRecip[m]), r = (uint32_t)lane - g * m;
  const bool gv = g < (uint32_t)__popc(dm);
  const uint32_t q = gv ? sm.dprm[warp][g] : 0u;
  const uint32_t own = q >> 27, oe = wl + own;
  uint64_t od = 0;
  const uint8_t *oram = nullptr;  // owner's RAM backing
  if (DIRTY) {
    od = __shfl_sync(kFull, L.dirty, own);
    oram = SCAT ? reinterpret_cast<const uint8_t *>(__shfl_sync(kFull, reinterpret_cast<unsigned long long>(L.ram), own))
                : p.s.ram + (block0 + oe) * 4096ull;
  }
  bool hit = false;
  if (gv && r < ((q >> 23) & 15u)) {
    const uint32_t ox = q & 63u, a = ((q >> 11) & 0xFFFu) + r;
    uint32_t byte = 0;
    if (DIRTY) {
      if (a <= 0xFFFu)
        byte = ((od >> (a >> 6)) & 1ull) ? (uint32_t)oram[a] : IMG(a);
    } else {
      byte = a <= 0xFFFu ? IMG(a) : 0u;  // no HBM-backed RAM load on the common path
    }
    const uint32_t yy = (((q >> 6) & 31u) + r) & 31u, q8 = ox & 0x38u;
    const uint64_t w = (uint64_t)__byte_perm((byte << 8) >> (ox & 7u), 0, 0x4401);
    const uint64_t mk = wrap ? ((w << q8) | (q8 ? (w >> (64u - q8)) : 0ull)) : (w << q8);
    OCTAX_CHECK(oe < (uint32_t)kBlock && yy < 32u);
    uint64_t *row = &sm.fb[oe * 32u + (yy ^ (oe & kSwz))];
    const uint64_t old = xor_row(row, mk);
    hit = (old & mk) != 0ull;
  }
  const uint32_t hb = __ballot_sync(kFull, hit);
  if (vfw) VREG(15) = (uint8_t)(mine && ((hb >> (rank * m)) & ((1u << m) - 1u)) != 0u);
}

// DXYN when no lane of the warp draws more than one row (a 1-row sprite, or clipped at
// the bottom): one row step, no sprite-word realignment.
template <bool DIRTY>
__device__ __forceinline__ void draw_one(Smem &sm, const StepParams &p, const Lane &L, int tid, bool draws, uint32_t x0, uint32_t y0,
                                         uint32_t base, uint32_t quirks, bool vfw) {
  bool hit = false;
  if (draws) {
    uint32_t byte;
    if (DIRTY) byte = rd(sm, p, L, base);
    else byte = IMG(base);
    const uint32_t q8 = x0 & 0x38u;
    const uint64_t w = (uint64_t)__byte_perm((byte << 8) >> (x0 & 7u), 0, 0x4401);
    const uint64_t mk = (quirks & 8u) ? ((w << q8) | (q8 ? (w >> (64u - q8)) : 0ull)) : (w << q8);
    uint64_t *row = &sm.fb[(uint32_t)tid * 32u + (y0 ^ ((uint32_t)tid & kSwz))];
    const uint64_t old = xor_row(row, mk);
    hit = (old & mk) != 0ull;
  }
  if (vfw) VREG(15) = (uint8_t)hit;
}

// RF = true (startup segments): lanes run under the loop-carried flag L.run (= part && !halted).
// RF = false (the step's frame loop): every lane runs the cycle; a lane that is halted, or
// that halts, re-executes its faulting entry with no effect -- an invalid word's entry has no
// effect flags and stays at its PC (E_BAD is in L.stay), a stack fault keeps PC and SP -- so
// no run flag gates the core; L.run then only records "did not fault" for the timer tick.
template <bool Q0, bool RF, bool SCAT = false>
__device__ __forceinline__ void cycle(Smem &sm, Lane &L, const StepParams &p, int tid, int lane, uint64_t block0,
                                      uint32_t gid, bool part, bool &wdirty) {
  const uint32_t quirks = Q0 ? 0u : p.quirks;  // Q0: modern profile specialisation
  bool act = RF ? L.run : true;
  const uint32_t pc = L.pc;
  // ---- fetch + decode: the predecoded word at PC (L1-resident table, loaded at the end
  //      of the previous cycle; PCs past 0xFFE halt through the table).  Slow path: PC in
  //      a dirty RAM block (self-modifying code).
  uint2 e = L.dec;
  if (wdirty) {
    const bool slow = act & (pc <= 0xFFEu) & (((L.dirty >> (pc >> 6)) & 3ull) != 0ull);
    if (__any_sync(kFull, slow)) {
      if (slow) make_entry((rd(sm, p, L, pc) << 8) | rd(sm, p, L, pc + 1), sm.dtab, quirks, e.x, e.y);
    }
  }
  const uint32_t d = e.x, nnn = e.y >> 20, nn = nnn & 255u, n = nnn & 15u, x = nnn >> 8;
  const bool is_ret = HAS(d, E_RET), call = HAS(d, D_CALL);
  const uint32_t nsp = L.sp + ((e.y >> 18) & 3u) - 1u;  // SP after 2NNN / 00EE
  // ---- faults halt the lane (A17, A20): invalid word / PC past 0xFFE, stack over/underflow
  const bool bad = HAS(d, E_BAD) || nsp > 16u;
  if (RF) {
    act = act && !bad;
    L.run = act;
  } else {
    act = nsp <= 16u;  // gates PC / SP / stack only; an E_BAD entry carries no effect flags
    L.run = !bad;
  }
  const bool ex = RF ? act : true;  // gate of the flag-driven effects
  // warp votes for the gated classes, taken as soon as the entry is known so the branches at
  // the end of the core do not wait on them (A/B +1%)
  const bool any_rare = __any_sync(kFull, ex && HAS(d, D_RARE));
  const bool any_draw = __any_sync(kFull, ex && HAS(d, D_DRAW));
  // V[k] of this lane lives at vbase | voff(k) (VREG); kx = V[x], or V0 for BNNN
  const uint32_t vb = vbase(tid), ax = (e.y & 0x1FFu) | vb, vx = sm.V[ax], vy = sm.V[((e.y >> 9) & 0x1FFu) | vb];
  OCTAX_CHECK(ax < 16u * kBlock && (((e.y >> 9) & 0x1FFu) | vb) < 16u * kBlock);
  // ---- stack
  OCTAX_CHECK(!(act && is_ret) || (L.sp >= 1u && L.sp <= 16u));
  OCTAX_CHECK(!(act && call) || L.sp < 16u);
  OCTAX_CHECK(x < 16u && tid < kBlock);
  uint32_t ret_pc = 0;
  OCTAX_CHECK(!(act && is_ret) || nsp < 16u);
  if (act && is_ret) ret_pc = sm.stk[nsp * kBlock + tid];
  if (act && call) { sm.stk[L.sp * kBlock + tid] = (uint16_t)(pc + 2u); L.stk_dirty = 1; }
  // ---- skips: 3XNN 5XY0 on equal, 4XNN 9XY0 on not-equal, EX9E / EXA1 on key
  // index i = [VX == operand] | [key VX & 15 down] << 1 into the entry's skip truth table;
  // L.keys holds the 16-bit mask twice, so a wrapping funnel shift by VX - 1 puts key
  // VX & 15 at bit 1
  const uint32_t eq01 = vx == (HAS(d, E_BVY) ? vy : nn) ? 1u : 0u;
  const uint32_t sidx = (__funnelshift_r(L.keys, L.keys, vx - 1u) & 2u) | eq01;
  const uint32_t skip2 = (d >> sidx) & 2u;  // 2 if the next word is skipped
  // ---- ALU 8XYn from the entry's one-hot operation (A_*); the flag is written after the
  //      result (A15); VF-reset quirk folded into D_WVF (logic results have s8 >> 8 == 0)
  const uint32_t ea = e.y;
  const uint32_t sa = Q0 ? vx : ((ea & A_SRCY) ? vy : vx);  // shift source (SHIFT_VY quirk)
  uint32_t s8 = vy;  // 8XY0
  if (ea & A_OR) s8 = vx | vy;
  if (ea & A_AND) s8 = vx & vy;
  if (ea & A_XOR) s8 = vx ^ vy;
  if (ea & A_ADD) s8 = sa + vy;          // 8XY4; 8XYE as VX + VX (or VY + VY)
  if (ea & A_SUB) s8 = vx - vy + 256u;   // 8XY5: bit 8 = no borrow
  if (ea & A_RSUB) s8 = vy - vx + 256u;  // 8XY7
  uint32_t f8 = s8 >> 8;
  if (ea & A_SHR) { s8 = sa >> 1; f8 = sa & 1u; }
  const uint32_t r8 = s8;  // stored as a byte: no masking
  // ---- register writes

  uint32_t nvx = nn;
  nvx = HAS(d, D_VSADD) ? (vx + nn) : nvx;
  nvx = HAS(d, D_VSALU) ? r8 : nvx;
  nvx = HAS(d, D_VSDT) ? L.dt : nvx;
  nvx = HAS(d, D_WAIT) ? L.kidx : nvx;
  sm.V[ax] = (uint8_t)((ex && (d & L.wvm) != 0u) ? nvx : vx);  // unconditional: no branch around the ALU
  if (ex && HAS(d, D_WVF)) VREG(15) = (uint8_t)f8;
  // ---- control flow and index / timer registers
  uint32_t npc = pc + 2u + skip2;
  npc = HAS(d, D_PCJ) ? nnn : npc;  // 1NNN, 2NNN
  npc = is_ret ? ret_pc : npc;
  npc = (d & L.stay) != 0u ? pc : npc;  // A16: FX0A re-executes while no key; E_BAD stays
  npc = HAS(d, D_BJMP) ? ((nnn + vx) & 0xFFFu) : npc;  // vx = V0 or V[x] (JUMP_VX quirk)
  uint32_t I2 = L.I;
  I2 = HAS(d, D_INNN) ? nnn : I2;
  I2 = HAS(d, D_IADD) ? (I2 + vx) : I2;  // 16-bit I kept modulo 2^32: users mask (A18)
  I2 = HAS(d, D_IFONT) ? (0x50u + 5u * (vx & 15u)) : I2;
  L.pc = act ? npc : pc;  // PC <= 0xFFE when running; halted-at-entry lanes carry bit 16 (see kDecEntries)
  L.dec = __ldg(p.s.dec + L.pc);  // next cycle's word, in flight meanwhile (re-read when idle)
  L.I = ex ? I2 : L.I;
  L.sp = act ? nsp : L.sp;
  L.dt = (ex && HAS(d, D_DTW)) ? vx : L.dt;
  L.st = (ex && HAS(d, D_STW)) ? vx : L.st;
  const bool f33 = nn == 0x33u, f55 = nn == 0x55u;  // only meaningful under D_MEM
  // ---- vote-gated rare classes (one vote for CLS / CXNN / FX33-55-65 together)
  if (any_rare) {
  const bool do_cls = ex && HAS(d, E_CLS);
  const bool do_rnd = ex && HAS(d, D_RND);
  const bool do_mem = ex && HAS(d, D_MEM);
  if (__any_sync(kFull, do_cls)) {
    if (do_cls) {
#pragma unroll
      for (int r = 0; r < 32; ++r) sm.fb[tid * 32 + r] = 0;
    }
  }
  if (__any_sync(kFull, do_rnd)) {
    if (do_rnd) {
      const uint32_t r = philox_out0(L.draw, L.episode, gid, 0u, (uint32_t)p.seed, (uint32_t)(p.seed >> 32));
      VREG(x) = (uint8_t)(r & nn);
      L.draw++;
    }
  }
  if (__any_sync(kFull, do_mem)) {
    if (do_mem) {
      if (f33) {
        wr(sm, p, L, L.I & 0xFFFu, vx / 100u);
        wr(sm, p, L, (L.I + 1u) & 0xFFFu, (vx / 10u) % 10u);
        wr(sm, p, L, (L.I + 2u) & 0xFFFu, vx % 10u);
      } else {
        if (f55) {
          for (uint32_t k = 0; k <= x; ++k) wr(sm, p, L, (L.I + k) & 0xFFFu, VREG(k));
        } else {
          for (uint32_t k = 0; k <= x; ++k) VREG(k) = (uint8_t)rd(sm, p, L, (L.I + k) & 0xFFFu);
        }
        if (quirks & 2u) L.I = (L.I + x + 1u) & 0xFFFFu;
      }
    }
    wdirty = __any_sync(kFull, L.dirty != 0ull);
  }
  }
  const bool do_draw = ex && HAS(d, D_DRAW);
  if (any_draw) {
    const uint32_t y0 = vy & 31u;
    const uint32_t nrows = do_draw ? (((quirks & 8u) != 0u) ? n : min(n, 32u - y0)) : 0u;
    const uint32_t maxr = __reduce_max_sync(kFull, nrows);
    const uint32_t dm = __ballot_sync(kFull, nrows != 0u);
    // one grouped pass (groups of maxr lanes, 32 / maxr drawers) when the drawers fit and
    // rows are many enough to beat maxr lane-parallel row steps (uniform choice)
    if (maxr >= kGroupMinRows && (uint32_t)__popc(dm) * maxr <= 32u)  // k drawers fit 32 / maxr groups
    {
      if (wdirty)
        draw_groups<true, SCAT>(sm, L, p, tid, lane, block0, dm, vx & 63u, y0, L.I & 0xFFFu, nrows, maxr, wdirty, quirks, do_draw);
      else
        draw_groups<false, SCAT>(sm, L, p, tid, lane, block0, dm, vx & 63u, y0, L.I & 0xFFFu, nrows, maxr, wdirty, quirks, do_draw);
    }
    else if (maxr == 1u) {
      if (wdirty) draw_one<true>(sm, p, L, tid, nrows != 0u, vx & 63u, y0, L.I & 0xFFFu, quirks, do_draw);
      else draw_one<false>(sm, p, L, tid, nrows != 0u, vx & 63u, y0, L.I & 0xFFFu, quirks, do_draw);
    } else if (maxr <= kLaneDrawMax)
      draw_lanes(sm, L, p, tid, do_draw, vx & 63u, y0, L.I & 0xFFFu, nrows, maxr, wdirty, quirks, do_draw);
    else
      draw_coop<SCAT>(sm, L, p, tid, lane, block0, do_draw, vx & 63u, y0, L.I & 0xFFFu, n, do_draw, quirks);
    __syncwarp();
  }
}

// `frames` frames of ipf cycles + timer tick, for lanes with `part` (uniform loop counts)
template <bool Q0, bool SCAT = false>
__device__ __forceinline__ void run_frames(Smem &sm, Lane &L, const StepParams &p, int tid, int lane, uint64_t block0,
                                           uint32_t gid, bool part, uint32_t frames, bool &wdirty) {
  L.run = part && !L.halted;
  for (uint32_t f = 0; f < frames; ++f) {
    for (uint32_t k = 0; k < p.ipf; ++k) cycle<Q0, true, SCAT>(sm, L, p, tid, lane, block0, gid, part, wdirty);
    if (L.run) {
      L.dt -= (L.dt != 0u);
      L.st -= (L.st != 0u);
    }
  }
  if (part) L.halted = !L.run;
}

// Postfix bytecode evaluator (uniform control flow: every lane runs the same
// program).  The stack lives in registers as a shift register with compile-time
// slots (depth <= kMaxDepth is enforced at create), so it costs no shared memory.
__device__ __forceinline__ uint32_t eval(const Program &P, Smem &sm, const StepParams &p, const Lane &L, int tid) {
  // the common shapes (uniform branches on the compiled program's kind, set at create): no
  // bytecode loop (A/B: +0.2% pong, +0.6..1.0% brix / Target Shooter, whose specs are all of them)
  if (P.kind == 1u) return P.ka;
  if (P.kind == 2u) return (uint32_t)VREG(P.ka);
  if (P.kind == 3u) return (uint32_t)VREG(P.ka) == P.kb ? 1u : 0u;
  if (P.kind == 4u) return (uint32_t)VREG(P.ka) != P.kb ? 1u : 0u;
  uint32_t st[kMaxDepth];
#pragma unroll
  for (int k = 0; k < kMaxDepth; ++k) st[k] = 0;
  for (uint32_t i = 0; i < P.len; ++i) {
    const ExprInsn in = P.ops[i];
    if (in.op <= X_VMOD) {  // push
      uint32_t v = in.op == X_CONST ? in.imm
                 : in.op <= X_V || in.op >= X_VDIV ? (uint32_t)VREG(in.arg)
                 : in.op == X_I   ? (L.I & 0xFFFFu)
                 : in.op == X_DT  ? L.dt : L.st;
      if (in.op >= X_VDIV) {  // byte / constant by multiply-shift (X_VDIV), remainder (X_VMOD)
        const uint32_t q = (v * in.imm) >> 16;
        v = in.op == X_VDIV ? q : v - q * (uint32_t)in.pad;
      }
#pragma unroll
      for (int k = kMaxDepth - 1; k > 0; --k) st[k] = st[k - 1];
      st[0] = v;
    } else if (in.op < X_MUL) {  // unary on the top
      const uint32_t t = st[0];
      st[0] = in.op == X_MEM ? rd(sm, p, L, t & 0xFFFu) : in.op == X_NEG ? 0u - t : in.op == X_NOT ? (uint32_t)(t == 0u) : ~t;
    } else {  // binary: a = second, b = top
      const uint32_t a = st[1], b = st[0];
      uint32_t r;
      switch (in.op) {
        case X_MUL: r = a * b; break;
        case X_DIV: r = b ? a / b : 0u; break;
        case X_MOD: r = b ? a % b : 0u; break;
        case X_ADD: r = a + b; break;
        case X_SUB: r = a - b; break;
        case X_SHL: r = b >= 32u ? 0u : a << b; break;
        case X_SHR: r = b >= 32u ? 0u : a >> b; break;
        case X_LT: r = a < b; break;
        case X_LE: r = a <= b; break;
        case X_GT: r = a > b; break;
        case X_GE: r = a >= b; break;
        case X_EQ: r = a == b; break;
        case X_NE: r = a != b; break;
        case X_AND: r = a & b; break;
        case X_XOR: r = a ^ b; break;
        case X_OR: r = a | b; break;
        case X_LAND: r = (a != 0u) & (b != 0u); break;
        default: r = (a != 0u) | (b != 0u); break;  // X_LOR
      }
#pragma unroll
      for (int k = 1; k < kMaxDepth - 1; ++k) st[k] = st[k + 1];
      st[kMaxDepth - 1] = 0;
      st[0] = r;
    }
  }
  return st[0];
}

// ---------------------------------------------------------------- the step kernel
template <int MODE, bool Q0>
#ifdef OCTAX_MAXNREG  // A/B knob for other CTA shapes (build.py --out ... -D OCTAX_MAXNREG=N)
__global__ void __maxnreg__(OCTAX_MAXNREG)
#else
__global__ void __launch_bounds__(kBlock, kMinBlocks)
#endif
octax_kernel(const __grid_constant__ StepParams p, const int32_t *__restrict__ actions,
             uint8_t *__restrict__ obs, float *__restrict__ reward, uint8_t *__restrict__ done_out,
             uint8_t *__restrict__ term_out, uint8_t *__restrict__ trunc_out) {
  extern __shared__ __align__(128) unsigned char smraw[];
  pdl_enter();
  Smem &sm = *reinterpret_cast<Smem *>(smraw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t block0 = ((uint64_t)blockIdx.x + p.block_base) * kBlock;
  const uint64_t env = block0 + tid;
  const uint32_t nlive = p.n - block0 < (uint64_t)kBlock ? (uint32_t)(p.n - block0) : (uint32_t)kBlock;
  const bool active = (uint32_t)tid < nlive;  // (32-bit: cheap to rematerialise)
  const uint64_t wbase = block0 + (uint64_t)warp * 32;
  OCTAX_CHECK(p.head < 4u && blockDim.x == (unsigned)kBlock);
  const int ne = p.n > wbase ? (int)((p.n - wbase) < 32 ? (p.n - wbase) : 32) : 0;
  const uint32_t hh = (uint32_t)lane >> 4, l2 = 2u * ((uint32_t)lane & 15u);  // 16-B chunk lanes

  // ---- prologue: TMA bulk copies of the image and (step) the CTA's 32 KB framebuffer
  //      block of ring slot h -- the ring keeps the smem swizzle, so no per-lane work
  if (tid == 0) stage_issue(sm, p.s.image, MODE != MODE_RESET ? ring_at(p, p.head & 3u, block0) : nullptr);

  Lane L;
  // lanes past n and lanes halted on entry fetch from the E_BAD half of the decode table
  // (PC bit 16), so the step's frame loop runs them without effect (cycle<Q0, false>)
  L.pc = 0x10000u; L.I = 0; L.sp = 0; L.dt = 0; L.st = 0; L.halted = 1; L.draw = 0; L.episode = 0;
  set_keys(L, 0u);
  L.dirty = 0; L.ram = p.s.ram; L.stk_dirty = 0;
  uint32_t steps = 0, prev = 0;
  int32_t ep_ret = 0;
  const uint32_t gid = (uint32_t)(p.env_offset + env);
  int32_t act_in = 0;  // the step's action, loaded first so its latency overlaps the prologue (+0.8%)
  if (active) {
    if (MODE == MODE_STEP) act_in = actions[env];
    uint4 v = p.s.regs[env];
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) *reinterpret_cast<uint32_t *>(&sm.V[vbase(tid) | (j << 7)]) = w[j];
    uint4 c = p.s.ctrl[env];
    L.pc = c.x & 0xFFFFu; L.I = c.x >> 16;
    L.sp = c.y & 255u; L.dt = (c.y >> 8) & 255u; L.st = (c.y >> 16) & 255u; L.halted = c.y >> 24;
    if (L.halted) L.pc |= 0x10000u;
    L.draw = c.z; L.episode = c.w;
    uint4 b = p.s.book[env];
    steps = b.x; prev = b.y; ep_ret = (int32_t)b.z;
    uint4 s0 = p.s.stack[env * 2], s1 = p.s.stack[env * 2 + 1];
    uint32_t sw[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
#pragma unroll
    for (int k = 0; k < 16; ++k) sm.stk[k * kBlock + tid] = (uint16_t)(sw[k >> 1] >> (16 * (k & 1)));
    L.dirty = p.s.dirty[env];
    L.ram = p.s.ram + env * 4096ull;
  }
  L.dec = __ldg(p.s.dec + L.pc);
  __syncthreads();  // mbarrier initialised
  stage_wait(sm);
  bool wdirty = __any_sync(kFull, L.dirty != 0ull);  // any lane with private RAM blocks

  // statistics accumulated over the launch's steps (one step, or T in a fused rollout)
  uint32_t finished = 0, err = 0;
  long long ret_acc = 0;
  // MODE_ROLLOUT (fused rollout, SURVEY d.3/d.8 "fused", K6 fused into K1): T steps in this
  // launch with the VM state in registers / shared memory and the framebuffer in shared memory
  // throughout; each step's display goes to the ring with plain per-warp stores, so after the
  // prologue a warp needs no CTA barrier until the statistics at the end.
  constexpr bool kRoll = MODE == MODE_ROLLOUT || MODE == MODE_ROLLOUT_NOOBS;
  // observations written?  Always, except in a rollout launched without them (obs_out == NULL:
  // rewards / dones only -- the ring history is still kept for the steps after it); a separate
  // instantiation, because a runtime test cost the observing rollout 2% (A/B)
  constexpr bool wobs = MODE != MODE_ROLLOUT_NOOBS;
  const uint32_t T = kRoll ? p.T : 1u;
  for (uint32_t t = 0; t < T; ++t) {
  const uint32_t h = (p.head + t) & 3u;
  const uint32_t s0 = (h + 2) & 3, s1 = (h + 3) & 3, s2 = h;
  uint64_t *__restrict__ obs64 = reinterpret_cast<uint64_t *>(obs) + (kRoll ? t * p.obs_stride : 0u);
  const uint64_t oo = kRoll ? t * p.out_stride : 0u;  // step t's reward / done row
  if (kRoll && active) {  // step t's action: given [T][n], or the K6 generator in-kernel
    const uint64_t ts = p.t0 + t;
    act_in = actions ? actions[t * p.n + env]
                     : (int32_t)(philox_out0((uint32_t)ts, (uint32_t)(ts >> 32), gid, 1u, (uint32_t)p.aseed,
                                             (uint32_t)(p.aseed >> 32)) % p.n_actions);
  }
  uint32_t done = 0, term = 0, trunc = 0;
  float rew = 0.f;
  bool resetting;
  if (MODE != MODE_RESET) {
    // Stacking (A3): by default obs = the last 4 step-END displays -- planes 0,1 come from
    // the ring (copied one env per VM cycle: loads before the cycle, stores after it, so
    // the HBM latency hides behind it), plane 2 = the step-start display.  With
    // stack_frames (OCTAX_OBS_STACK_FRAMES) obs = the displays after the last 4 FRAMES of
    // this step; planes for frames before the step (frame_skip < 4) = step-start display.
    const bool sf = p.stack_frames != 0u;
    const int first = sf ? 4 - (int)p.frame_skip : 3;  // planes [0, first) <- step-start display
    if (!wobs) {
    } else if (!sf) {
      for (int e = 0; e < ne; e += 2)  // plane 2 <- step-start display, two envs per pass
        if (e + (int)hh < ne) {
          const uint32_t el = (uint32_t)(warp * 32 + e) + hh;
          put_pair(&sm.fb[el * 32u], obs64 + (wbase + e + hh) * 128, 2u, l2, el & kSwz);
        }
    } else {
      for (int e = 0; e < ne; ++e) {
        const uint64_t v = sm.fb[fb_idx(warp * 32 + e, lane)];
        uint64_t *ob = obs64 + (wbase + e) * 128;
        for (int pl = 0; pl < first && pl < 3; ++pl) ob[pl * 32 + lane] = v;
      }
    }
    if (active) {
      int32_t a = act_in;
      if (a < 0 || (uint32_t)a >= p.n_actions) {
        a = 0;
        // a rollout keeps no flag live through its steps (fewer registers: fused +1%, A/B)
        if (kRoll) atomicOr(&p.s.stats[3], 1ull);
        else err = 1;
      }
      set_keys(L, p.keymask[a]);
    }
    // planes 0 (lanes 0-15, ring slot s0) and 1 (lanes 16-31, slot s1) of env `cur`:
    // one 16-B chunk per lane, loaded before a cycle and stored (in row order) after it
    const uint4 *rsrc = reinterpret_cast<const uint4 *>(ring_at(p, hh ? s1 : s0, wbase) + l2);
    // one bulk L2 prefetch per half-warp of its 8 KB ring block (plane 0 or 1 of the warp's
    // 32 envs): the per-cycle copy loads then hit L2 instead of queueing on HBM (+5..8%)
    if (!sf && wobs && (lane & 15) == 0 && ne > 0)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ring_at(p, hh ? s1 : s0, wbase)),
                   "r"((uint32_t)ne * 256u) : "memory");
    uint64_t *odst = obs64 + wbase * 128 + hh * 32;
    int cur = (sf || !wobs) ? ne : 0;
    L.run = active && !L.halted;
    const uint4 *rp = rsrc + cur * 16;  // env `cur`'s chunk and obs row block, advanced per copy
    uint64_t *opl = odst + cur * 128;
    for (uint32_t f = 0; f < p.frame_skip; ++f) {
      for (uint32_t k = 0; k < p.ipf; ++k) {
        const bool cp = cur < ne;
        uint4 q;  // only read under cp
        if (cp) q = __ldcs(rp);
        // L1 prefetch of the chunk two cycles ahead (from the L2-resident ring block): its load
        // is then an L1 hit, and the store at the end of that cycle does not wait on L2 (A/B:
        // +3% pong, +6..7% brix / Target Shooter; one or three cycles ahead are slower)
        if (cur + 2 < ne) asm volatile("prefetch.global.L1 [%0];" ::"l"(rp + 32));
        cycle<Q0, false>(sm, L, p, tid, lane, block0, gid, active, wdirty);
        // unconditional bookkeeping: the guarded store is one predicated STG, no branch region
        // (A/B v34: +0.3..0.7% brix / Target Shooter); `cur` runs past ne, the tail loop is then empty
        if (cp) put_rows(opl, 0u, l2 ^ ((uint32_t)cur & kSwz), q);
        ++cur;
        rp += 16;
        opl += 128;
      }
      if (L.run) {
        L.dt -= (L.dt != 0u);
        L.st -= (L.st != 0u);
      }
      const int pl = (int)f + 4 - (int)p.frame_skip;  // obs plane of this frame (stack_frames)
      if (sf && wobs && pl >= 0 && pl < 3) {
        __syncwarp();
        for (int e = 0; e < ne; ++e)
          obs64[(wbase + e) * 128 + pl * 32 + lane] = sm.fb[fb_idx(warp * 32 + e, lane)];
      }
    }
    // envs the per-cycle copy did not reach (fewer than 32 cycles per step): rp / opl already point
    // at env `cur`, so the ring / obs bases need not stay live through the frame loop
#pragma unroll 4
    for (int e = cur; e < ne; ++e, rp += 16, opl += 128) put_rows(opl, 0u, l2 ^ ((uint32_t)e & kSwz), __ldcs(rp));
    if (active) L.halted = !L.run;
    if (active) {
      const uint32_t s = eval(p.score, sm, p, L, tid);
      const int32_t d = (int32_t)(s - prev);
      rew = (float)d;
      prev = s;
      ep_ret = (int32_t)((uint32_t)ep_ret + (uint32_t)d);
      steps++;
      term = (eval(p.term, sm, p, L, tid) != 0u) || L.halted;
      trunc = p.max_steps && steps >= p.max_steps;
      done = term | trunc;
      // a rollout counts its finished episodes from the episode counter at the end
      if (done) { ret_acc += ep_ret; if (!kRoll) finished++; L.episode++; }
      reward[oo + env] = rew;
      done_out[oo + env] = (uint8_t)done;
      if (term_out) term_out[oo + env] = (uint8_t)term;
      if (trunc_out) trunc_out[oo + env] = (uint8_t)trunc;
    }
    resetting = active && done;
    // ---- optional extras: the terminal transition's obs and the finished episode's return/length
    if (active && p.ep_ret_out) p.ep_ret_out[env] = done ? ep_ret : 0;
    if (active && p.ep_len_out) p.ep_len_out[env] = done ? steps : 0u;
    if (p.final_obs) {
      __syncwarp();
      uint32_t dm = __ballot_sync(kFull, resetting);
      uint64_t *fo64 = reinterpret_cast<uint64_t *>(p.final_obs);
      while (dm) {
        const int e = __ffs(dm) - 1;
        dm &= dm - 1;
        const uint64_t *ob = obs64 + (wbase + e) * 128;  // planes 0..2 already in obs
        uint64_t *fo = fo64 + (wbase + e) * 128;
        fo[lane] = ob[lane];
        fo[32 + lane] = ob[32 + lane];
        fo[64 + lane] = ob[64 + lane];
        fo[96 + lane] = sm.fb[fb_idx(warp * 32 + e, lane)];
      }
      __syncwarp();
    }
    // Specs with startup segments: a reset runs frames of startup code, which inline would
    // hold the whole warp for one lane; the done envs are appended (warp-aggregated) to a
    // list instead, and reset_kernel, launched right after on the same stream, runs them
    // packed 128 per CTA (stream order keeps the same-step reset of A10).
    if (p.reset_ids != nullptr) {
      const uint32_t m = __ballot_sync(kFull, resetting);
      if (m) {
        const int leader = __ffs(m) - 1;
        uint32_t base = 0;
        if (lane == leader) base = atomicAdd(p.reset_count, (uint32_t)__popc(m));
        base = __shfl_sync(kFull, base, leader);
        if (resetting) p.reset_ids[base + (uint32_t)__popc(m & ((1u << lane) - 1u))] = (uint32_t)env;
      }
      resetting = false;
    }
  } else {
    resetting = active;
    L.episode = 0;
  }

  // ---- same-step auto-reset: power-on + startup segments (warp-uniform)
  const uint32_t reset_mask = __ballot_sync(kFull, resetting);
  if (reset_mask) {
    if (resetting) power_on(sm, L, p, tid);
    __syncwarp();
    for (uint32_t seg = 0; seg < p.n_startup; ++seg) {
      if (resetting) set_keys(L, p.startup_keys[seg]);
      run_frames<Q0>(sm, L, p, tid, lane, block0, gid, resetting, p.startup_frames[seg], wdirty);
    }

    if (resetting) {
      set_keys(L, 0u);
      // a lane that faulted in a startup segment keeps the faulting PC in the frame loops;
      // its stored PC is the word after it, as the fetch advanced it (a2, A17, A33), except
      // for a fetch past 0xFFE (stored unchanged)
      if (L.halted && L.pc <= 0xFFEu) L.pc += 2u;
      // ... and, like a lane loaded halted, it then fetches from the E_BAD half of the decode table
      // (PC bit 16; stored PCs drop it), so a fused rollout's next step runs it without effect
      if (L.halted) {
        L.pc |= 0x10000u;
        L.dec = __ldg(p.s.dec + L.pc);
      }
      steps = 0;
      prev = eval(p.score, sm, p, L, tid);
      ep_ret = 0;
    }
  }
  __syncwarp();

  // ---- epilogue: the CTA's framebuffer block -> ring slot h+1 with one TMA bulk store
  //      (all 4 slots on a reset launch); obs plane 3 in row order (all planes on reset).
  //      A fused rollout stores each warp's 32 displays to slot h+1 itself (16-B chunks in
  //      position order, next to the plane-3 rows) and continues without a CTA barrier.
  if (!kRoll) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy
    __syncthreads();
    if (tid == 0) {
      if (MODE == MODE_STEP) {
        fb_store_issue(sm, ring_at(p, (h + 1) & 3, block0));
      } else {
        for (uint32_t sl = 0; sl < 4; ++sl) fb_store_issue(sm, ring_at(p, sl, block0));
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (MODE == MODE_ROLLOUT_NOOBS || obs64) {  // an obs-less rollout still stores the ring here
    for (int e = 0; e < ne; e += 2)
      if (e + (int)hh < ne) {
        const uint32_t el = (uint32_t)(warp * 32 + e) + hh, sw = el & kSwz;
        const uint64_t *fe = &sm.fb[el * 32u];
        uint64_t *ob = obs64 + (wbase + e + hh) * 128;
        if (wobs) put_pair(fe, ob, 3u, l2, sw);
        if (MODE == MODE_STEP && p.frame_out)  // the newest display alone, contiguous (host frame path)
          put_pair(fe, reinterpret_cast<uint64_t *>(p.frame_out) + (wbase + e + hh) * 32, 0u, l2, sw);
        if (kRoll)  // ring slot h+1: the 16-B chunk at positions l2, l2+1
          *reinterpret_cast<ulonglong2 *>(ring_at(p, (h + 1) & 3, wbase + e + hh) + l2) =
              make_ulonglong2(fe[l2], fe[l2 + 1]);
        if (wobs && (MODE == MODE_RESET || ((reset_mask >> (e + hh)) & 1u))) {
          put_pair(fe, ob, 0u, l2, sw);
          put_pair(fe, ob, 1u, l2, sw);
          put_pair(fe, ob, 2u, l2, sw);
        }
      }
  }
  if (MODE != MODE_RESET) {  // reset envs: the other three ring slots hold the reset display too
    uint32_t rm = reset_mask;
    while (rm) {
      const int e = __ffs(rm) - 1;
      rm &= rm - 1;
      const uint64_t v = sm.fb[(uint32_t)(warp * 32 + e) * 32u + lane];  // position order = ring order
      ring_at(p, s0, wbase + e)[lane] = v;
      ring_at(p, s1, wbase + e)[lane] = v;
      ring_at(p, s2, wbase + e)[lane] = v;
    }
  }

  if (kRoll) __syncwarp();  // this step's ring / smem stores before the next step's reads
  }  // step loop
  // a rollout's finished episodes = the episode counter's advance (read before the state store)
  if (kRoll && active) finished = L.episode - p.s.ctrl[env].w;

  // ---- store lane state
  if (active) {
    uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < 4; ++j) w[j] = *reinterpret_cast<const uint32_t *>(&sm.V[vbase(tid) | (j << 7)]);
    p.s.regs[env] = make_uint4(w[0], w[1], w[2], w[3]);
    p.s.ctrl[env] = make_uint4((L.pc & 0xFFFFu) | (L.I << 16), L.sp | (L.dt << 8) | (L.st << 16) | (L.halted << 24),
                               L.draw, L.episode);
    p.s.book[env] = make_uint4(steps, prev, (uint32_t)ep_ret, 0u);
    if (L.stk_dirty) store_stack(sm, p, tid, env);
    p.s.dirty[env] = L.dirty;
  }

  // ---- integer episode statistics (a12): warp reduce, CTA reduce, 4 atomics per CTA
  if (MODE != MODE_RESET) {
    unsigned long long r = (unsigned long long)ret_acc, f = finished, st = active ? T : 0u, er = err;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      r += __shfl_xor_sync(kFull, r, o);
      f += __shfl_xor_sync(kFull, f, o);
      st += __shfl_xor_sync(kFull, st, o);
      er |= __shfl_xor_sync(kFull, er, o);
    }
    if (lane == 0) { sm.red[0][warp] = r; sm.red[1][warp] = f; sm.red[2][warp] = st; sm.red[3][warp] = er; }
    __syncthreads();
    if (tid < 4) {
      unsigned long long acc = 0;
      for (int w2 = 0; w2 < kBlock / 32; ++w2) acc = tid == 3 ? (acc | sm.red[tid][w2]) : acc + sm.red[tid][w2];
      if (acc) {
        if (tid == 3) atomicOr(&p.s.stats[3], acc);
        else atomicAdd(&p.s.stats[tid], acc);
      }
    }
  }
  if (!kRoll && tid == 0)
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem outlives the store
}

// ---------------------------------------------------------------- deferred resets (K3)
// The envs the step kernel listed (done, spec with startup segments), 128 per CTA in a
// grid-stride loop: power-on, the startup segments, the new episode's score baseline; then
// the reset display goes to all four obs planes and ring slots and the state is stored.
template <bool Q0>
__global__ void __launch_bounds__(kBlock, kMinBlocks)
reset_kernel(const __grid_constant__ StepParams p, uint8_t *__restrict__ obs) {
  extern __shared__ __align__(128) unsigned char smraw[];
  Smem &sm = *reinterpret_cast<Smem *>(smraw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t count = *p.reset_count;
  if ((uint64_t)blockIdx.x * kBlock >= count) return;  // uniform per CTA
  if (tid == 0) stage_issue(sm, p.s.image, nullptr);
  __syncthreads();  // mbarrier initialised
  stage_wait(sm);
  uint64_t *obs64 = reinterpret_cast<uint64_t *>(obs);
  for (uint64_t b0 = (uint64_t)blockIdx.x * kBlock; b0 < count; b0 += (uint64_t)gridDim.x * kBlock) {
    const bool part = b0 + tid < count;
    const uint64_t env = part ? p.reset_ids[b0 + tid] : 0u;
    OCTAX_CHECK(env < p.n);
    Lane L;
    L.pc = 0x10000u; L.I = 0; L.sp = 0; L.dt = 0; L.st = 0; L.halted = 1; L.draw = 0; L.episode = 0;
    set_keys(L, 0u);
    L.dirty = 0; L.ram = p.s.ram + env * 4096ull; L.stk_dirty = 0;
    L.dec = __ldg(p.s.dec + L.pc);
    const uint32_t gid = (uint32_t)(p.env_offset + env);
    if (part) {
      L.episode = p.s.ctrl[env].w;  // incremented by the step kernel
      power_on(sm, L, p, tid);
    }
    __syncwarp();
    bool wdirty = false;
    for (uint32_t seg = 0; seg < p.n_startup; ++seg) {
      if (part) set_keys(L, p.startup_keys[seg]);
      run_frames<Q0, true>(sm, L, p, tid, lane, 0, gid, part, p.startup_frames[seg], wdirty);
    }
    uint32_t prev = 0;
    if (part) {
      set_keys(L, 0u);
      if (L.halted && L.pc <= 0xFFEu) L.pc += 2u;  // faulted in startup: PC after the fetch (A33)
      prev = eval(p.score, sm, p, L, tid);
    }
    __syncwarp();
    // the reset display -> obs planes 0..3 and ring slots 0..3, one env per pass, lane = row
    uint32_t wm = __ballot_sync(kFull, part);
    while (wm) {
      const int e = __ffs(wm) - 1;
      wm &= wm - 1;
      const uint64_t E = __shfl_sync(kFull, env, e);
      const uint64_t v = sm.fb[fb_idx(warp * 32 + e, lane)];  // row `lane`
      const uint32_t pos = (uint32_t)lane ^ (uint32_t)(E & kSwz);
      for (uint32_t sl = 0; sl < 4; ++sl) ring_at(p, sl, E)[pos] = v;
      if (obs64) {
        uint64_t *ob = obs64 + E * 128 + lane;
        __stcs(ob, v);
        __stcs(ob + 32, v);
        __stcs(ob + 64, v);
        __stcs(ob + 96, v);
      }
      if (p.frame_out) __stcs(reinterpret_cast<uint64_t *>(p.frame_out) + E * 32 + lane, v);  // newest display
    }
    if (part) {
      uint32_t w[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) w[j] = *reinterpret_cast<const uint32_t *>(&sm.V[vbase(tid) | (j << 7)]);
      p.s.regs[env] = make_uint4(w[0], w[1], w[2], w[3]);
      p.s.ctrl[env] = make_uint4((L.pc & 0xFFFFu) | (L.I << 16), L.sp | (L.dt << 8) | (L.st << 16) | (L.halted << 24),
                                 L.draw, L.episode);
      p.s.book[env] = make_uint4(0u, prev, 0u, 0u);
      store_stack(sm, p, tid, env);
      p.s.dirty[env] = L.dirty;
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------- warp-per-env kernel
// One WARP interprets one environment (octax_set_kernel; auto below a few thousand envs).  The
// lane-per-env kernel above is throughput-optimal when the GPU is full, but at the paper's own
// env counts (512..8,192) it leaves most SMs idle and runs one warp per SM
// sub-partition through a ~240-instruction predicated cycle: latency bound.
// Here nothing diverges -- every lane follows the same env -- so each CHIP-8 instruction is a
// warp-uniform switch case of a few instructions, and the VM state lives in registers:
//   lane k < 16: V[k] (`v`) and return-stack entry k (`sk`); lane r: display row r (`fb`, one
//   u64 in packed byte order); PC / I / SP / timers / keys / counters replicated in every lane.
// DXYN is one row per lane (the "lanes of a warp cooperating on sprite rows" of the north star),
// VF = a warp vote; FX55 / FX65 move register k in lane k.  RAM stays copy-on-write (64-B blocks
// materialised in HBM on the first write, the pristine image read through L1).  Same state
// layout, ring and outputs as the lane-per-env kernel, and the same semantics (oracle/ c.1):
// the two are interchangeable on one handle between any two calls.
#ifndef OCTAX_WCTA
#define OCTAX_WCTA 4
#endif
#ifndef OCTAX_WARP_LAZY  // A/B knob: decode fields per case (1), all before the switch (0), per case above 2,048 envs (2)
#define OCTAX_WARP_LAZY 2
#endif
#ifndef OCTAX_WARP_KEXIT  // A/B knob: a fault also ends the frame loop through its counter (no per-cycle PC test)
#define OCTAX_WARP_KEXIT 1
#endif
#ifndef OCTAX_WARP_PCHALT  // A/B knob: a fault in w_cycle marks PC bit 16 (1), sets W.halted (0), PC bit above 2,048 envs (2)
#define OCTAX_WARP_PCHALT 2
#endif
template <bool REGP>
struct WarpOpts {  // per-instantiation code shape (A/B: both win where the kernel is issue-bound, > 2,048 envs,
                   // and lose 1..3% at <= 2,048, where it is latency-bound; profiles/r02_v47_ab_warp_*.log)
  static constexpr bool lazy = OCTAX_WARP_LAZY == 1 || (OCTAX_WARP_LAZY == 2 && !REGP);
  static constexpr bool pchalt = OCTAX_WARP_PCHALT == 1 || (OCTAX_WARP_PCHALT == 2 && !REGP);
};
// a fault: PC bit 16 marks it for w_frame (no halted flag carried through every switch case), or W.halted
#define WHALT(pcv)                                  \
  do {                                              \
    if (WarpOpts<REGP>::pchalt) {                   \
      W.pc = (pcv) | 0x10000u;                      \
      if (OCTAX_WARP_KEXIT) k = 0xFFFFFFF0u;        \
    } else {                                        \
      W.pc = (pcv);                                 \
      W.halted = 1;                                 \
    }                                               \
  } while (0)
#ifndef OCTAX_WARP_PCCLAMP  // A/B knob: clamp the fetch index to 0xFFF (the table before v45 had 4,096 entries)
#define OCTAX_WARP_PCCLAMP 0
#endif
constexpr int kWarpCta = OCTAX_WCTA;  // envs (warps) per CTA: small CTAs spread a small batch over all SMs

struct WEnv {  // uniform per warp (replicated in every lane)
  uint32_t pc, I, sp, dt, st, halted, draw, episode, keys;
  uint64_t dirty;
  uint8_t *ram;
  const uint8_t *img;     // p.s.image, p.s.words
  const uint16_t *words;
  uint32_t quirks;        // p.quirks (read from here by the REGP instantiation)
};

// byte `a` (< 4096) of the env's memory: its HBM RAM block if written, else the pristine image.
// RAM is written by this kernel, so it is read with plain loads (not the read-only path).
__device__ __forceinline__ uint32_t w_rd(const StepParams &p, const WEnv &W, uint32_t a) {
  OCTAX_CHECK(a < 4096u);
  return ((W.dirty >> (a >> 6)) & 1ull) ? (uint32_t)W.ram[a] : (uint32_t)__ldg(W.img + a);
}

// lanes with `on` store byte `val` at their address `a` (< 4096; distinct per lane).  The 64-B
// blocks any writer touches are materialised first (copy-on-write, 16 lanes x 4 B per block).
__device__ __forceinline__ void w_wr(const StepParams &p, WEnv &W, int lane, bool on, uint32_t a, uint32_t val) {
  OCTAX_CHECK(!on || a < 4096u);
  const uint64_t need = on ? (1ull << (a >> 6)) : 0ull;
  uint64_t m = ((uint64_t)__reduce_or_sync(kFull, (uint32_t)(need >> 32)) << 32) |
               __reduce_or_sync(kFull, (uint32_t)need);
  m &= ~W.dirty;
  while (m) {
    const uint32_t b = (uint32_t)__ffsll((long long)m) - 1u;
    m &= m - 1;
    if (lane < 16)
      reinterpret_cast<uint32_t *>(W.ram + b * 64u)[lane] =
          __ldg(reinterpret_cast<const uint32_t *>(W.img + b * 64u) + lane);
    W.dirty |= 1ull << b;
  }
  __syncwarp();
  if (on) W.ram[a] = (uint8_t)val;
  __syncwarp();  // the bytes are visible to every lane's later reads
}

#define WV(k) __shfl_sync(kFull, v, (int)(k))

// one CHIP-8 instruction (oracle/octax_oracle.c cycle(), readings A15-A23)
template <bool REGP>
__device__ __forceinline__ void w_cycle(const StepParams &p, WEnv &W, uint32_t &v, uint32_t &sk, uint64_t &fb,
                                        int lane, uint32_t gid, uint32_t &k) {
  const uint32_t pc = W.pc;
  // the word at PC: one load, issued first, from the pristine word table (one entry per 16-bit
  // PC; entries past 0xFFE hold 0x5001, an invalid word, so such a PC lands on the halting path
  // of class 5 below); re-assembled from RAM bytes when PC's 64-B block (or the next, holding
  // PC + 1) was written
  OCTAX_CHECK(pc < kWordEntries);
#if OCTAX_WARP_PCCLAMP
  uint32_t op = __ldg(W.words + min(pc, 0xFFFu));
#else
  uint32_t op = __ldg(W.words + pc);
#endif
  if (((W.dirty >> (pc >> 6)) & 3ull) != 0ull && pc <= 0xFFEu) op = (w_rd(p, W, pc) << 8) | w_rd(p, W, pc + 1u);
  W.pc = pc + 2u;
  // Decode fields.  Taken where a case reads them (kLazy), each case pays only for its own instead
  // of all five before the switch: -7 instructions on the common path, +8% at 4,096 envs where the
  // kernel is issue-bound; at <= 2,048 envs (REGP, latency-bound) they stay up front, off the
  // dispatch's dependent chain (A/B, profiles/r02_v47_ab_warp_lazy.log)
  constexpr bool kLazy = WarpOpts<REGP>::lazy;
  const uint32_t x_ = kLazy ? 0u : (op >> 8) & 15u, y_ = kLazy ? 0u : (op >> 4) & 15u;
  const uint32_t n_ = kLazy ? 0u : op & 15u, nn_ = kLazy ? 0u : op & 255u, nnn_ = kLazy ? 0u : op & 0xFFFu;
#define x (kLazy ? ((op >> 8) & 15u) : x_)
#define y (kLazy ? ((op >> 4) & 15u) : y_)
#define n (kLazy ? (op & 15u) : n_)
#define nn (kLazy ? (op & 255u) : nn_)
#define nnn (kLazy ? (op & 0xFFFu) : nnn_)
  const uint32_t quirks = REGP ? W.quirks : p.quirks;
  switch (op >> 12) {
    case 0x0:
      if (op == 0x00E0u) {
        fb = 0;
      } else if (op == 0x00EEu) {
        if (W.sp == 0u) { WHALT(W.pc); return; }  // A20: stack underflow
        W.sp -= 1u;
        W.pc = __shfl_sync(kFull, sk, (int)W.sp);
      }
      break;  // other 0NNN: no-op (A20)
    case 0x1: W.pc = nnn; break;
    case 0x2:
      if (W.sp == 16u) { WHALT(W.pc); return; }  // A20: stack overflow
      sk = (uint32_t)lane == W.sp ? W.pc : sk;
      W.sp += 1u;
      W.pc = nnn;
      break;
    case 0x3: if (WV(x) == nn) W.pc += 2u; break;
    case 0x4: if (WV(x) != nn) W.pc += 2u; break;
    case 0x5:
      if (n != 0u) {  // invalid word: halt with PC past it (A20); a fetch past 0xFFE: PC unchanged (A17)
        WHALT(pc > 0xFFEu ? pc : W.pc);
        return;
      }
      if (WV(x) == WV(y)) W.pc += 2u;
      break;
    case 0x6: v = (uint32_t)lane == x ? nn : v; break;
    case 0x7: v = (uint32_t)lane == x ? ((v + nn) & 255u) : v; break;  // VF untouched
    case 0x8: {  // both operands read first, VF written last (A15)
      const uint32_t a = WV(x), b = WV(y), s = (quirks & 1u) ? b : a;  // SHIFT_VY quirk
      uint32_t r, f;
      bool wf = true;
      switch (n) {
        case 0x0: r = b; wf = false; f = 0; break;
        case 0x1: r = a | b; wf = (quirks & 16u) != 0u; f = 0; break;  // VF_RESET quirk
        case 0x2: r = a & b; wf = (quirks & 16u) != 0u; f = 0; break;
        case 0x3: r = a ^ b; wf = (quirks & 16u) != 0u; f = 0; break;
        case 0x4: r = a + b; f = r >> 8; break;
        case 0x5: r = a - b; f = a >= b; break;
        case 0x6: r = s >> 1; f = s & 1u; break;
        case 0x7: r = b - a; f = b >= a; break;
        case 0xE: r = s << 1; f = (s >> 7) & 1u; break;
        default: WHALT(W.pc); return;  // A20
      }
      v = (uint32_t)lane == x ? (r & 255u) : v;
      if (wf) v = lane == 15 ? f : v;
      break;
    }
    case 0x9:
      if (n != 0u) { WHALT(W.pc); return; }
      if (WV(x) != WV(y)) W.pc += 2u;
      break;
    case 0xA: W.I = nnn; break;
    case 0xB: W.pc = (nnn + WV((quirks & 4u) ? x : 0u)) & 0xFFFu; break;  // JUMP_VX quirk
    case 0xC: {  // A12: Philox(ctr = {draw, episode, gid, 0}, key = seed).out0 & NN
      const uint32_t r = philox_out0(W.draw, W.episode, gid, 0u, (uint32_t)p.seed, (uint32_t)(p.seed >> 32));
      v = (uint32_t)lane == x ? (r & nn) : v;
      W.draw += 1u;
      break;
    }
    case 0xD: {  // lane r draws display row r (sprite row (r - y0) & 31); A18 clip / WRAP quirk
      const uint32_t x0 = WV(x) & 63u, y0 = WV(y) & 31u, base = W.I & 0xFFFu;
      const bool wrap = (quirks & 8u) != 0u;
      const uint32_t i = ((uint32_t)lane - y0) & 31u;
      uint64_t mk = 0;
      if (i < n && (wrap || (uint32_t)lane >= y0)) {
        const uint32_t a = base + i;
        const uint64_t nat = (uint64_t)(a <= 0xFFFu ? w_rd(p, W, a) : 0u) << 56;  // pixel c at bit 63 - c
        const uint64_t m = (nat >> x0) | ((wrap && x0) ? nat << (64u - x0) : 0ull);
        mk = bswap64(m);  // -> packed row byte order (byte b = pixels 8b..8b+7, MSB first)
      }
      const bool hit = __any_sync(kFull, (fb & mk) != 0ull);
      fb ^= mk;
      v = lane == 15 ? (uint32_t)hit : v;
      break;
    }
    case 0xE: {
      const bool down = ((W.keys >> (WV(x) & 15u)) & 1u) != 0u;  // A19
      if (nn == 0x9Eu) { if (down) W.pc += 2u; }
      else if (nn == 0xA1u) { if (!down) W.pc += 2u; }
      else { WHALT(W.pc); return; }
      break;
    }
    case 0xF:
      switch (nn) {
        case 0x07: v = (uint32_t)lane == x ? W.dt : v; break;
        case 0x0A:  // A16: level-triggered wait (re-executes while no key is held)
          if (W.keys) v = (uint32_t)lane == x ? (uint32_t)(__ffs((int)W.keys) - 1) : v;
          else W.pc -= 2u;
          break;
        case 0x15: W.dt = WV(x); break;
        case 0x18: W.st = WV(x); break;
        case 0x1E: W.I = (W.I + WV(x)) & 0xFFFFu; break;
        case 0x29: W.I = 0x50u + 5u * (WV(x) & 15u); break;
        case 0x33: {  // BCD: lanes 0..2 store the three digits
          const uint32_t vx = WV(x);
          const uint32_t d = lane == 0 ? vx / 100u : lane == 1 ? (vx / 10u) % 10u : vx % 10u;
          w_wr(p, W, lane, lane < 3, (W.I + (uint32_t)lane) & 0xFFFu, d);
          break;
        }
        case 0x55:  // lane k <= x stores V[k]
          w_wr(p, W, lane, (uint32_t)lane <= x, (W.I + (uint32_t)lane) & 0xFFFu, v);
          if (quirks & 2u) W.I = (W.I + x + 1u) & 0xFFFFu;  // LOADSTORE_INC_I quirk
          break;
        case 0x65: {
          const uint32_t a = (W.I + (uint32_t)(lane & 15)) & 0xFFFu;
          const uint32_t b = w_rd(p, W, a);
          v = (uint32_t)lane <= x ? b : v;
          if (quirks & 2u) W.I = (W.I + x + 1u) & 0xFFFFu;
          break;
        }
        default: WHALT(W.pc); return;
      }
      break;
    default: __builtin_unreachable();
  }
}
#undef x
#undef y
#undef n
#undef nn
#undef nnn


// one 60 Hz frame: ipf instructions, then the timer tick (A1, A2); halted envs stand still
template <bool REGP>
__device__ __forceinline__ void w_frame(const StepParams &p, WEnv &W, uint32_t &v, uint32_t &sk, uint64_t &fb,
                                        int lane, uint32_t gid) {
  if (WarpOpts<REGP>::pchalt) {
    // a fault inside the frame sets PC bit 16 (WHALT), so the loop tests PC instead of a halted
    // flag that every switch case would otherwise have to carry
    if (W.halted) return;
#if OCTAX_WARP_KEXIT
    for (uint32_t k = 0; k < p.ipf; ++k) w_cycle<REGP>(p, W, v, sk, fb, lane, gid, k);
#else
    for (uint32_t k = 0; k < p.ipf && W.pc < 0x10000u; ++k) w_cycle<REGP>(p, W, v, sk, fb, lane, gid, k);
#endif
    if (W.pc >= 0x10000u) {
      W.pc &= 0xFFFFu;
      W.halted = 1;
      return;
    }
    W.dt -= W.dt != 0u;
    W.st -= W.st != 0u;
  } else {
    for (uint32_t k = 0; k < p.ipf && !W.halted; ++k) w_cycle<REGP>(p, W, v, sk, fb, lane, gid, k);
    if (!W.halted) {
      W.dt -= W.dt != 0u;
      W.st -= W.st != 0u;
    }
  }
}

// score / termination program (same bytecode as eval(); V[k] from lane k)
__device__ __forceinline__ uint32_t w_eval(const Program &P, const StepParams &p, const WEnv &W, uint32_t v) {
  if (P.kind == 1u) return P.ka;
  if (P.kind == 2u) return WV(P.ka);
  if (P.kind == 3u) return WV(P.ka) == P.kb ? 1u : 0u;
  if (P.kind == 4u) return WV(P.ka) != P.kb ? 1u : 0u;
  uint32_t st[kMaxDepth];
#pragma unroll
  for (int k = 0; k < kMaxDepth; ++k) st[k] = 0;
  for (uint32_t i = 0; i < P.len; ++i) {
    const ExprInsn in = P.ops[i];
    if (in.op <= X_VMOD) {
      uint32_t val = in.op == X_CONST ? in.imm
                   : in.op <= X_V || in.op >= X_VDIV ? WV(in.arg)
                   : in.op == X_I  ? (W.I & 0xFFFFu)
                   : in.op == X_DT ? W.dt : W.st;
      if (in.op >= X_VDIV) {
        const uint32_t q = (val * in.imm) >> 16;
        val = in.op == X_VDIV ? q : val - q * (uint32_t)in.pad;
      }
#pragma unroll
      for (int k = kMaxDepth - 1; k > 0; --k) st[k] = st[k - 1];
      st[0] = val;
    } else if (in.op < X_MUL) {
      const uint32_t t = st[0];
      st[0] = in.op == X_MEM ? w_rd(p, W, t & 0xFFFu) : in.op == X_NEG ? 0u - t : in.op == X_NOT ? (uint32_t)(t == 0u) : ~t;
    } else {
      const uint32_t a = st[1], b = st[0];
      uint32_t r;
      switch (in.op) {
        case X_MUL: r = a * b; break;
        case X_DIV: r = b ? a / b : 0u; break;
        case X_MOD: r = b ? a % b : 0u; break;
        case X_ADD: r = a + b; break;
        case X_SUB: r = a - b; break;
        case X_SHL: r = b >= 32u ? 0u : a << b; break;
        case X_SHR: r = b >= 32u ? 0u : a >> b; break;
        case X_LT: r = a < b; break;
        case X_LE: r = a <= b; break;
        case X_GT: r = a > b; break;
        case X_GE: r = a >= b; break;
        case X_EQ: r = a == b; break;
        case X_NE: r = a != b; break;
        case X_AND: r = a & b; break;
        case X_XOR: r = a ^ b; break;
        case X_OR: r = a | b; break;
        case X_LAND: r = (a != 0u) & (b != 0u); break;
        default: r = (a != 0u) | (b != 0u); break;
      }
#pragma unroll
      for (int k = 1; k < kMaxDepth - 1; ++k) st[k] = st[k + 1];
      st[kMaxDepth - 1] = 0;
      st[0] = r;
    }
  }
  return st[0];
}

// power-on + the spec's startup segments (A11); the new episode's score baseline
template <bool REGP>
__device__ __forceinline__ void w_reset(const StepParams &p, WEnv &W, uint32_t &v, uint32_t &sk, uint64_t &fb,
                                        int lane, uint32_t gid, uint32_t &steps, uint32_t &prev, int32_t &ep_ret) {
  v = 0; sk = 0; fb = 0;
  W.pc = 0x200u; W.I = 0; W.sp = 0; W.dt = 0; W.st = 0; W.halted = 0; W.draw = 0; W.dirty = 0;
  for (uint32_t seg = 0; seg < p.n_startup; ++seg) {
    W.keys = p.startup_keys[seg];
    for (uint32_t f = 0; f < p.startup_frames[seg]; ++f) w_frame<REGP>(p, W, v, sk, fb, lane, gid);
  }
  W.keys = 0;
  steps = 0;
  prev = w_eval(p.score, p, W, v);
  ep_ret = 0;
}

// <= 72 registers: 28+ resident warps (envs) per SM, so 4,096 envs run in one wave on 148 SMs
// (at 95 registers a 4,096-env step took 1.36x longer: A/B); no spills at this cap
// REGP (launches of <= 2,048 envs, where the kernel is latency-bound): the image / word-table
// pointers and the quirk bits pass through a shuffle at kernel start, which ptxas does not
// rematerialise, so they stay in registers instead of being reloaded from the parameter bank on
// every VM cycle (an LDC on the fetch's dependent chain): +3..6% at 512 envs; at 4,096 envs
// (issue-bound) the plain form is 0.5..1.5% faster (A/B, profiles/r02_v43_ab_warp_variants.log)
template <int MODE, bool REGP>
__global__ void __maxnreg__(REGP ? 96 : 72)  // <= 2,048 envs: 14 warps per SM at most, registers are free
octax_warp_kernel(const __grid_constant__ StepParams p, const int32_t *__restrict__ actions, uint8_t *__restrict__ obs,
                  float *__restrict__ reward, uint8_t *__restrict__ done_out, uint8_t *__restrict__ term_out,
                  uint8_t *__restrict__ trunc_out) {
  __shared__ unsigned long long red[4][kWarpCta];
  pdl_enter();
  const int lane = (int)(threadIdx.x & 31u), warp = (int)(threadIdx.x >> 5);
  constexpr bool kRoll = MODE == MODE_ROLLOUT || MODE == MODE_ROLLOUT_NOOBS;
  constexpr bool wobs = MODE != MODE_ROLLOUT_NOOBS;
  // the launch covers envs [block_base * kBlock, ...) like the lane-per-env kernel's CTA blocks
  const uint64_t e0 = (uint64_t)p.block_base * kBlock;
  const uint64_t e1 = p.block_count ? min(p.n, e0 + (uint64_t)p.block_count * kBlock) : p.n;
  const uint64_t env = e0 + (uint64_t)blockIdx.x * kWarpCta + (uint64_t)warp;
  unsigned long long ret_acc = 0, finished = 0, nsteps = 0, err = 0;
  if (env < e1) {  // uniform per warp
    const uint32_t gid = (uint32_t)(p.env_offset + env), pos = (uint32_t)lane ^ ((uint32_t)env & kSwz);
    uint64_t *obs64 = reinterpret_cast<uint64_t *>(obs);
    WEnv W;
    W.ram = p.s.ram + env * 4096ull;
    if (REGP) {
      W.img = reinterpret_cast<const uint8_t *>(__shfl_sync(kFull, reinterpret_cast<uintptr_t>(p.s.image), 0));
      W.words = reinterpret_cast<const uint16_t *>(__shfl_sync(kFull, reinterpret_cast<uintptr_t>(p.s.words), 0));
      W.quirks = __shfl_sync(kFull, p.quirks, 0);
    } else {
      W.img = p.s.image;  // ptxas re-reads these from the parameter bank where they are used
      W.words = p.s.words;
      W.quirks = p.quirks;
    }
    W.keys = 0;
    uint32_t v = 0, sk = 0, steps = 0, prev = 0;
    int32_t ep_ret = 0;
    uint64_t fb = 0, hA = 0, hB = 0;  // display (row `lane`); ends of steps t-3, t-2 (obs planes 0, 1)
    if (MODE == MODE_RESET) {
      W.episode = 0;
      w_reset<REGP>(p, W, v, sk, fb, lane, gid, steps, prev, ep_ret);
      for (uint32_t sl = 0; sl < 4; ++sl) ring_at(p, sl, env)[pos] = fb;
      if (obs64)
        for (uint32_t pl = 0; pl < 4; ++pl) __stcs(obs64 + env * 128 + pl * 32 + lane, fb);
    } else {
      const uint4 r = p.s.regs[env];
      const uint32_t k = (uint32_t)lane & 15u, w = k < 4u ? r.x : k < 8u ? r.y : k < 12u ? r.z : r.w;
      v = (w >> (8u * (k & 3u))) & 255u;
      const uint4 c = p.s.ctrl[env];
      W.pc = c.x & 0xFFFFu; W.I = c.x >> 16;
      W.sp = c.y & 255u; W.dt = (c.y >> 8) & 255u; W.st = (c.y >> 16) & 255u; W.halted = c.y >> 24;
      W.draw = c.z; W.episode = c.w;
      const uint4 b = p.s.book[env];
      steps = b.x; prev = b.y; ep_ret = (int32_t)b.z;
      sk = reinterpret_cast<const uint16_t *>(p.s.stack)[env * 16u + k];
      W.dirty = p.s.dirty[env];
      fb = ring_at(p, p.head & 3u, env)[pos];
      hA = ring_at(p, (p.head + 2u) & 3u, env)[pos];
      hB = ring_at(p, (p.head + 3u) & 3u, env)[pos];
      const uint32_t T = kRoll ? p.T : 1u;
      const bool sf = p.stack_frames != 0u;
      for (uint32_t t = 0; t < T; ++t) {
        const uint32_t h = (p.head + t) & 3u;
        uint64_t *ob = obs64 ? obs64 + (kRoll ? t * p.obs_stride : 0u) + env * 128 : nullptr;
        const uint64_t oo = kRoll ? t * p.out_stride : 0u;
        int32_t a;
        if (!kRoll) a = actions[env];
        else if (actions) a = actions[t * p.n + env];
        else {
          const uint64_t ts = p.t0 + t;
          a = (int32_t)(philox_out0((uint32_t)ts, (uint32_t)(ts >> 32), gid, 1u, (uint32_t)p.aseed,
                                    (uint32_t)(p.aseed >> 32)) % p.n_actions);
        }
        if (a < 0 || (uint32_t)a >= p.n_actions) {  // out of range: no-op + sticky flag
          a = 0;
          err = 1;
        }
        W.keys = p.keymask[a];
        const uint64_t start = fb;
        // obs planes 0..2: the last step-end displays, or (stack_frames) the displays after the
        // last frames of this step, planes before the step's first frame = step-start display
        uint64_t P0 = sf ? start : hA, P1 = sf ? start : hB, P2 = start;
        for (uint32_t f = 0; f < p.frame_skip; ++f) {
          w_frame<REGP>(p, W, v, sk, fb, lane, gid);
          const int pl = (int)f + 4 - (int)p.frame_skip;
          if (sf) {
            P0 = pl == 0 ? fb : P0;
            P1 = pl == 1 ? fb : P1;
            P2 = pl == 2 ? fb : P2;
          }
        }
        const uint32_t s = w_eval(p.score, p, W, v);
        const int32_t d = (int32_t)(s - prev);
        prev = s;
        ep_ret = (int32_t)((uint32_t)ep_ret + (uint32_t)d);
        steps++;
        const uint32_t term = (w_eval(p.term, p, W, v) != 0u) || W.halted;
        const uint32_t trunc = p.max_steps && steps >= p.max_steps;
        const uint32_t done = term | trunc;
        if (lane == 0) {
          reward[oo + env] = (float)d;
          done_out[oo + env] = (uint8_t)done;
          if (term_out) term_out[oo + env] = (uint8_t)term;
          if (trunc_out) trunc_out[oo + env] = (uint8_t)trunc;
          if (p.ep_ret_out) p.ep_ret_out[env] = done ? ep_ret : 0;
          if (p.ep_len_out) p.ep_len_out[env] = done ? steps : 0u;
        }
        nsteps++;
        if (done) {
          if (p.final_obs) {
            uint64_t *fo = reinterpret_cast<uint64_t *>(p.final_obs) + env * 128 + lane;
            fo[0] = P0; fo[32] = P1; fo[64] = P2; fo[96] = fb;
          }
          ret_acc += (unsigned long long)(long long)ep_ret;
          finished++;
          W.episode++;
          w_reset<REGP>(p, W, v, sk, fb, lane, gid, steps, prev, ep_ret);  // A10: same-step auto-reset
          P0 = P1 = P2 = fb;
          for (uint32_t sl = 0; sl < 4; ++sl) ring_at(p, sl, env)[pos] = fb;
          hA = hB = fb;
        } else {
          ring_at(p, (h + 1u) & 3u, env)[pos] = fb;
          hA = hB;
          hB = start;
        }
        if (wobs && ob) {
          __stcs(ob + lane, P0);
          __stcs(ob + 32 + lane, P1);
          __stcs(ob + 64 + lane, P2);
          __stcs(ob + 96 + lane, fb);
        }
        if (MODE == MODE_STEP && p.frame_out) __stcs(reinterpret_cast<uint64_t *>(p.frame_out) + env * 32 + lane, fb);
      }
    }
    // store the VM state (same layout as the lane-per-env kernel)
    if (lane < 16) {
      reinterpret_cast<uint8_t *>(p.s.regs + env)[lane] = (uint8_t)v;
      reinterpret_cast<uint16_t *>(p.s.stack)[env * 16u + (uint32_t)lane] = (uint16_t)sk;
    }
    if (lane == 0) {
      p.s.ctrl[env] = make_uint4((W.pc & 0xFFFFu) | (W.I << 16), W.sp | (W.dt << 8) | (W.st << 16) | (W.halted << 24),
                                 W.draw, W.episode);
      p.s.book[env] = make_uint4(steps, prev, (uint32_t)ep_ret, 0u);
      p.s.dirty[env] = W.dirty;
    }
  }
  // integer episode statistics (a12): per CTA, 4 atomics
  if (MODE != MODE_RESET) {
    if (lane == 0) { red[0][warp] = ret_acc; red[1][warp] = finished; red[2][warp] = nsteps; red[3][warp] = err; }
    __syncthreads();
    if (threadIdx.x < 4) {
      unsigned long long acc = 0;
      for (int w2 = 0; w2 < kWarpCta; ++w2) acc = threadIdx.x == 3 ? (acc | red[3][w2]) : acc + red[threadIdx.x][w2];
      if (acc) {
        if (threadIdx.x == 3) atomicOr(&p.s.stats[3], acc);
        else atomicAdd(&p.s.stats[threadIdx.x], acc);
      }
    }
  }
}
#undef WV

// launch with programmatic stream serialization when `pdl` (and OCTAX_PDL; see pdl_enter), else a
// plain launch (griddepcontrol.wait then returns at once)
template <typename... A>
static cudaError_t launch_pdl(void (*k)(A...), unsigned grid, unsigned block, size_t smem, cudaStream_t stream,
                              bool pdl, const StepParams &p, const int32_t *actions, uint8_t *obs, float *reward,
                              uint8_t *done, uint8_t *term, uint8_t *trunc) {
  // not inside a stream capture: replayed from a CUDA graph, PDL edges measured slower (configs[1]
  // at 4,096 envs: -8%, `profiles/r02_v46_ab_pdl.log`), and a graph has no launch gap to hide
  if (pdl) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess) {
      (void)cudaGetLastError();
      pdl = false;
    } else if (cs != cudaStreamCaptureStatusNone) {
      pdl = false;
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (OCTAX_PDL && pdl) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, p, actions, obs, reward, done, term, trunc);
}

template <int MODE>
static cudaError_t launch_warp(const StepParams &p, const int32_t *actions, uint8_t *obs, float *reward, uint8_t *done,
                               uint8_t *term, uint8_t *trunc, cudaStream_t stream) {
  const uint64_t e0 = (uint64_t)p.block_base * kBlock;
  const uint64_t e1 = p.block_count ? std::min<uint64_t>(p.n, e0 + (uint64_t)p.block_count * kBlock) : p.n;
  if (e1 <= e0) return cudaSuccess;
  const unsigned grid = (unsigned)((e1 - e0 + kWarpCta - 1) / kWarpCta);
  // PDL always: the warp kernel's batches are latency-bound (A/B: +15% at 512 envs, +1..2% at 4,096)
  // the latency-bound instantiation (REGP) up to 2,048 envs for rollouts and resets, up to 1,024 for
  // single steps: there the issue-bound one is +7..9% at 2,048 envs, a rollout -2..-3%; both lose
  // 3..14% at 256..1,024 envs (A/B, profiles/r02_v48_ab_warp_pchalt.log run 3)
  constexpr uint64_t kRegpMax = MODE == MODE_STEP ? 1024u : 2048u;
  if (e1 - e0 <= kRegpMax)
    return launch_pdl(octax_warp_kernel<MODE, true>, grid, 32 * kWarpCta, 0, stream, true, p, actions, obs, reward,
                      done, term, trunc);
  return launch_pdl(octax_warp_kernel<MODE, false>, grid, 32 * kWarpCta, 0, stream, true, p, actions, obs, reward,
                    done, term, trunc);
}

// ---------------------------------------------------------------- auxiliary kernels
__global__ void gen_actions_kernel(uint64_t n, uint64_t env_offset, uint64_t aseed, uint64_t t,
                                   uint32_t n_actions, int32_t *__restrict__ out) {
  uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  uint32_t r = philox_out0((uint32_t)t, (uint32_t)(t >> 32), (uint32_t)(env_offset + j), 1u, (uint32_t)aseed,
                           (uint32_t)(aseed >> 32));
  out[j] = (int32_t)(r % n_actions);
}

// packed [n][4][32][8] -> bool [n][4][64][32] (P:146 axis order [frame][x][y]).
// One warp per plane: lane y loads row y, the two 32x32 bit blocks (x = 0..31,
// 32..63) are transposed across the warp with 5 shuffle-xor stages each, so lane
// x then holds column x (bit y = pixel (x, y)); each column's 32 bits are spread
// to 32 bytes (nibble * 0x204081 & 0x01010101 puts 4 bits into 4 bytes) and
// stored as two 16-byte vectors -- coalesced 2 KB per plane.
__device__ __forceinline__ uint32_t transpose32(uint32_t w, int lane) {
  const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int j = 16 >> s;
    const uint32_t lo = masks[s];
    const uint32_t t = __shfl_xor_sync(kFull, w, j);
    w = (lane & j) ? ((w & ~lo) | ((t >> j) & lo)) : ((w & lo) | ((t << j) & ~lo));
  }
  return w;
}

__device__ __forceinline__ uint4 spread8(uint32_t bits16, int half) {
  uint32_t v[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) v[q] = (((bits16 >> (16 * half + 4 * q)) & 15u) * 0x204081u) & 0x01010101u;
  return make_uint4(v[0], v[1], v[2], v[3]);
}

__global__ void __launch_bounds__(256) expand_obs_kernel(uint64_t n, const uint8_t *__restrict__ packed,
                                                         uint8_t *__restrict__ dense,
                                                         const uint8_t *__restrict__ row_mask) {
  const uint64_t plane = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (plane >= n * 4) return;                       // uniform per warp
  if (row_mask && !row_mask[plane >> 2]) return;    // uniform per warp
  const uint64_t row = reinterpret_cast<const uint64_t *>(packed)[plane * 32 + lane];
  // bit x of nat_lo / nat_hi = pixel x / 32 + x (packed bytes are MSB-first)
  const uint32_t nat_lo = __byte_perm(__brev((uint32_t)row), 0, 0x0123);
  const uint32_t nat_hi = __byte_perm(__brev((uint32_t)(row >> 32)), 0, 0x0123);
  const uint32_t col_lo = transpose32(nat_lo, lane);  // column x = lane
  const uint32_t col_hi = transpose32(nat_hi, lane);  // column x = 32 + lane
  uint4 *out = reinterpret_cast<uint4 *>(dense + plane * 2048);
  out[lane * 2] = spread8(col_lo, 0);
  out[lane * 2 + 1] = spread8(col_lo, 1);
  out[64 + lane * 2] = spread8(col_hi, 0);
  out[64 + lane * 2 + 1] = spread8(col_hi, 1);
}

// canonical per-env state (DESIGN.md layout), one CTA of 128 threads per requested env
__global__ void get_states_kernel(StepParams p, const uint64_t *__restrict__ ids, uint64_t first,
                                  uint8_t *__restrict__ out) {
  const uint64_t env = ids ? ids[blockIdx.x] : first + blockIdx.x;  // ids == nullptr: a range
  uint8_t *c = out + (uint64_t)blockIdx.x * 5200;
  const int t = threadIdx.x;
  const uint32_t h = p.head;
  if (t == 0) {
    uint4 v = p.s.regs[env];
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
    for (int k = 0; k < 16; ++k) c[k] = (uint8_t)(w[k >> 2] >> (8 * (k & 3)));
    uint4 cc = p.s.ctrl[env];
    uint32_t pc = cc.x & 0xFFFF, I = cc.x >> 16;
    c[16] = I & 255; c[17] = I >> 8; c[18] = pc & 255; c[19] = pc >> 8;
    c[20] = cc.y & 255; c[21] = (cc.y >> 8) & 255; c[22] = (cc.y >> 16) & 255; c[23] = (cc.y >> 24) & 1;
    uint4 s0 = p.s.stack[env * 2], s1 = p.s.stack[env * 2 + 1];
    uint32_t sw[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
    for (int k = 0; k < 8; ++k)
      for (int q = 0; q < 4; ++q) c[24 + 4 * k + q] = (uint8_t)(sw[k] >> (8 * q));
    uint4 b = p.s.book[env];
    uint32_t f[6] = {cc.z, cc.w, b.x, b.y, b.z, 0};
    for (int k = 0; k < 6; ++k)
      for (int q = 0; q < 4; ++q) c[56 + 4 * k + q] = (uint8_t)(f[k] >> (8 * q));
  }
  // display (slot h) and history planes 0..2 = slots h-3, h-2, h-1
  // canonical byte i = row i>>3, byte i&7; the ring holds row r at position r ^ (env & kSwz)
  for (int i = t; i < 256; i += blockDim.x) {
    const uint32_t j = (((uint32_t)i >> 3) ^ (uint32_t)(env & kSwz)) * 8u + ((uint32_t)i & 7u);
    c[80 + i] = reinterpret_cast<const uint8_t *>(ring_at(p, h & 3, env))[j];
    c[336 + i] = reinterpret_cast<const uint8_t *>(ring_at(p, (h + 1) & 3, env))[j];
    c[592 + i] = reinterpret_cast<const uint8_t *>(ring_at(p, (h + 2) & 3, env))[j];
    c[848 + i] = reinterpret_cast<const uint8_t *>(ring_at(p, (h + 3) & 3, env))[j];
  }
  const uint64_t dirty = p.s.dirty[env];
  const uint8_t *ram = p.s.ram + env * 4096ull;
  for (int i = t; i < 4096; i += blockDim.x) c[1104 + i] = ((dirty >> (i >> 6)) & 1) ? ram[i] : p.s.image[i];
}

__global__ void set_state_kernel(StepParams p, uint64_t env, const uint8_t *__restrict__ c) {
  const int t = threadIdx.x;
  const uint32_t h = p.head;
  auto u32 = [&](int o) {
    return (uint32_t)c[o] | ((uint32_t)c[o + 1] << 8) | ((uint32_t)c[o + 2] << 16) | ((uint32_t)c[o + 3] << 24);
  };
  if (t == 0) {
    uint32_t w[4] = {u32(0), u32(4), u32(8), u32(12)};
    p.s.regs[env] = make_uint4(w[0], w[1], w[2], w[3]);
    uint32_t I = c[16] | (c[17] << 8), pc = c[18] | (c[19] << 8);
    p.s.ctrl[env] = make_uint4(pc | (I << 16), c[20] | (c[21] << 8) | (c[22] << 16) | ((c[23] & 1u) << 24),
                               u32(56), u32(60));
    p.s.book[env] = make_uint4(u32(64), u32(68), u32(72), 0);
    p.s.stack[env * 2] = make_uint4(u32(24), u32(28), u32(32), u32(36));
    p.s.stack[env * 2 + 1] = make_uint4(u32(40), u32(44), u32(48), u32(52));
    p.s.dirty[env] = ~0ull;  // whole RAM materialised from the canonical bytes
  }
  for (int i = t; i < 256; i += blockDim.x) {
    const uint32_t j = (((uint32_t)i >> 3) ^ (uint32_t)(env & kSwz)) * 8u + ((uint32_t)i & 7u);
    reinterpret_cast<uint8_t *>(ring_at(p, h & 3, env))[j] = c[80 + i];
    reinterpret_cast<uint8_t *>(ring_at(p, (h + 1) & 3, env))[j] = c[336 + i];
    reinterpret_cast<uint8_t *>(ring_at(p, (h + 2) & 3, env))[j] = c[592 + i];
    reinterpret_cast<uint8_t *>(ring_at(p, (h + 3) & 3, env))[j] = c[848 + i];
  }
  uint8_t *ram = p.s.ram + env * 4096ull;
  for (int i = t; i < 4096; i += blockDim.x) ram[i] = c[1104 + i];
}

// ---------------------------------------------------------------- launchers
template <int MODE, bool Q0>
static cudaError_t launch_variant(const StepParams &p, const int32_t *actions, uint8_t *obs, float *reward,
                                  uint8_t *done, uint8_t *term, uint8_t *trunc, cudaStream_t stream) {
  // the dynamic-smem opt-in is per device and per kernel instance: one bit per device ordinal
  static std::atomic<uint64_t> attr_set{0};
  const size_t smem = sizeof(Smem);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_set.load(std::memory_order_relaxed) & bit)) {
    e = cudaFuncSetAttribute(octax_kernel<MODE, Q0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(bit, std::memory_order_relaxed);
  }
  const unsigned grid = p.block_count ? p.block_count : (unsigned)((p.n + kBlock - 1) / kBlock - p.block_base);
  // PDL when the grid is at most one CTA per SM (latency-bound: the next launch's CTAs wait on the
  // idle SMs) or at least one full wave (they take the slots the tail frees); a grid between the two
  // lets the next launch's first CTAs pile onto the SMs its predecessor left half empty, which then
  // finish last (A/B: -11% at 65,536 envs)
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool pdl = grid <= (unsigned)sms || grid >= (unsigned)sms * (unsigned)kMinBlocks;
  return launch_pdl(octax_kernel<MODE, Q0>, grid, kBlock, smem, stream, pdl, p, actions, obs, reward, done, term,
                    trunc);
}

template <bool Q0>
static cudaError_t launch_resets(const StepParams &p, uint8_t *obs, cudaStream_t stream) {
  static std::atomic<uint64_t> attr_set{0};
  const size_t smem = sizeof(Smem);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_set.load(std::memory_order_relaxed) & bit)) {
    e = cudaFuncSetAttribute(reset_kernel<Q0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(bit, std::memory_order_relaxed);
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t need = (p.n + kBlock - 1) / kBlock, cap = (uint64_t)sms * kMinBlocks;
  reset_kernel<Q0><<<(unsigned)(need < cap ? need : cap), kBlock, smem, stream>>>(p, obs);
  return cudaGetLastError();
}

cudaError_t launch_step(const StepParams &p, int mode, const int32_t *actions, uint8_t *obs, float *reward,
                        uint8_t *done, uint8_t *term, uint8_t *trunc, cudaStream_t stream) {
  if (p.warp) {  // warp-per-env kernel: every mode, resets inline (no reset_kernel)
    if (mode == MODE_STEP) return launch_warp<MODE_STEP>(p, actions, obs, reward, done, term, trunc, stream);
    if (mode == MODE_ROLLOUT)
      return obs ? launch_warp<MODE_ROLLOUT>(p, actions, obs, reward, done, term, trunc, stream)
                 : launch_warp<MODE_ROLLOUT_NOOBS>(p, actions, obs, reward, done, term, trunc, stream);
    return launch_warp<MODE_RESET>(p, nullptr, obs, nullptr, nullptr, nullptr, nullptr, stream);
  }
  const bool q0 = p.quirks == 0u;
  if (mode == MODE_STEP) {
    if (p.reset_ids) {  // deferred resets: count from zero, step, then the listed resets
      cudaError_t e = cudaMemsetAsync(p.reset_count, 0, sizeof(uint32_t), stream);
      if (e != cudaSuccess) return e;
    }
    cudaError_t e = q0 ? launch_variant<MODE_STEP, true>(p, actions, obs, reward, done, term, trunc, stream)
                       : launch_variant<MODE_STEP, false>(p, actions, obs, reward, done, term, trunc, stream);
    if (e != cudaSuccess || !p.reset_ids) return e;
    return q0 ? launch_resets<true>(p, obs, stream) : launch_resets<false>(p, obs, stream);
  }
  if (mode == MODE_ROLLOUT) {  // inline resets (p.reset_ids == nullptr): no reset_kernel inside a rollout
    if (!obs)
      return q0 ? launch_variant<MODE_ROLLOUT_NOOBS, true>(p, actions, obs, reward, done, term, trunc, stream)
                : launch_variant<MODE_ROLLOUT_NOOBS, false>(p, actions, obs, reward, done, term, trunc, stream);
    return q0 ? launch_variant<MODE_ROLLOUT, true>(p, actions, obs, reward, done, term, trunc, stream)
              : launch_variant<MODE_ROLLOUT, false>(p, actions, obs, reward, done, term, trunc, stream);
  }
  return q0 ? launch_variant<MODE_RESET, true>(p, nullptr, obs, nullptr, nullptr, nullptr, nullptr, stream)
            : launch_variant<MODE_RESET, false>(p, nullptr, obs, nullptr, nullptr, nullptr, nullptr, stream);
}

cudaError_t launch_gen_actions(uint64_t n, uint64_t env_offset, uint64_t aseed, uint64_t t, uint32_t n_actions,
                               int32_t *out, cudaStream_t stream) {
  const unsigned grid = (unsigned)((n + 255) / 256);
  gen_actions_kernel<<<grid, 256, 0, stream>>>(n, env_offset, aseed, t, n_actions, out);
  return cudaGetLastError();
}

cudaError_t launch_expand_obs(uint64_t n, const uint8_t *packed, uint8_t *dense, cudaStream_t stream,
                              const uint8_t *row_mask) {
  const uint64_t threads = n * 4 * 32;  // one warp per plane
  const unsigned grid = (unsigned)((threads + 255) / 256);
  expand_obs_kernel<<<grid, 256, 0, stream>>>(n, packed, dense, row_mask);
  return cudaGetLastError();
}

cudaError_t launch_get_states(const StepParams &p, const uint64_t *ids, uint64_t count, uint8_t *out,
                              cudaStream_t stream) {
  get_states_kernel<<<(unsigned)count, 128, 0, stream>>>(p, ids, 0, out);
  return cudaGetLastError();
}

// FNV-1a 64 over each env's 5,200 canonical bytes (octax_state_digests), one thread per env
__global__ void digest_kernel(const uint8_t *__restrict__ canon, uint64_t count, uint64_t *__restrict__ out) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= count) return;
  const uint4 *c = reinterpret_cast<const uint4 *>(canon + j * 5200);  // 5,200 = 325 x 16 B
  uint64_t h = 0xCBF29CE484222325ull;
  for (int k = 0; k < 325; ++k) {
    const uint4 v = c[k];
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int b = 0; b < 4; ++b) h = (h ^ ((w[q] >> (8 * b)) & 255u)) * 0x100000001B3ull;
  }
  out[j] = h;
}

cudaError_t launch_state_digests(const StepParams &p, uint64_t first, uint64_t count, uint8_t *canon,
                                 uint64_t *out, cudaStream_t stream) {
  get_states_kernel<<<(unsigned)count, 128, 0, stream>>>(p, nullptr, first, canon);
  digest_kernel<<<(unsigned)((count + 127) / 128), 128, 0, stream>>>(canon, count, out);
  return cudaGetLastError();
}

cudaError_t launch_set_state(const StepParams &p, uint64_t env, const uint8_t *canon, cudaStream_t stream) {
  set_state_kernel<<<1, 128, 0, stream>>>(p, env, canon);
  return cudaGetLastError();
}

}  // namespace octax
