// octax_kernels.cu -- sm_100a kernels of the batched Octax environment step.
//
// One thread = one environment (CHIP-8 VM), 128 envs per CTA.  Per step:
//   * the 4 KB pristine image (font + ROM) is staged once per CTA into shared
//     memory with a TMA bulk copy (cp.async.bulk + mbarrier);
//   * a warp-cooperative prologue streams the three previous display planes
//     of its 32 envs from the HBM ring straight into obs planes 0..2
//     (coalesced 256 B per env-plane) and the newest one into the shared-memory
//     framebuffer (32 x u64 rows per env, padded to 33 to stay bank-conflict
//     free);
//   * each lane interprets frame_skip x instructions_per_frame CHIP-8 cycles
//     (P:142-146), V0..VF in shared memory ([16][128] u32: any V[x] access by
//     any lane mix is conflict free), DXYN as 64-bit XOR row ops on the smem
//     framebuffer, RAM reads from the smem image unless the
//     64-B block is dirty (copy-on-write overlay in HBM);
//   * score / termination bytecode -> reward, done; same-step
//     auto-reset with startup segments (A10);
//   * a warp-cooperative epilogue writes obs plane 3 and the new ring slot;
//   * per-CTA integer episode statistics -> 4 int64 atomics per CTA.
// Semantics follow DESIGN.md readings A1..A27; nothing here is shared with
// the CPU oracle in oracle/.
#include <cuda_runtime.h>

#include <cstdint>

#include "octax_dev.cuh"

namespace octax {

struct __align__(128) Smem {
  uint8_t img[kImageBytes];                  // pristine image (TMA destination)
  uint64_t fb[kBlock * kFbStride];           // framebuffer rows, bit 63-x = pixel x
  uint32_t V[16 * kBlock];                   // V[k*kBlock + tid]
  uint16_t stk[16 * kBlock];                 // stk[k*kBlock + tid]
  uint32_t evs[kMaxDepth * kBlock];          // expression stack (below top)
  unsigned long long red[4][kBlock / 32];    // per-warp statistics
  unsigned long long bar;                    // mbarrier for the image copy
};

size_t smem_bytes() { return sizeof(Smem); }

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

// ---------------------------------------------------------------- TMA image load
__device__ __forceinline__ void image_load_issue(Smem &sm, const uint8_t *src) {
  uint32_t bar = (uint32_t)__cvta_generic_to_shared(&sm.bar);
  uint32_t dst = (uint32_t)__cvta_generic_to_shared(sm.img);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kImageBytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(kImageBytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void image_load_wait(Smem &sm) {
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

// ---------------------------------------------------------------- lane state
struct Lane {
  uint32_t pc, I, sp, dt, st, halted, keys, draw, episode;
  uint64_t dirty;
  uint8_t *ram;
  uint32_t stk_dirty;
};

#define VREG(k) sm.V[(k)*kBlock + tid]
#define FBROW(r) sm.fb[tid * kFbStride + (r)]

__device__ __forceinline__ uint32_t rd(const Smem &sm, const Lane &L, uint32_t a) {
  return ((L.dirty >> (a >> 6)) & 1ull) ? (uint32_t)L.ram[a] : (uint32_t)sm.img[a];
}

__device__ __forceinline__ void wr(const Smem &sm, Lane &L, uint32_t a, uint32_t v) {
  uint32_t b = a >> 6;
  if (!((L.dirty >> b) & 1ull)) {  // copy-on-write: materialise the 64-B block
    const uint4 *src = reinterpret_cast<const uint4 *>(sm.img + b * 64);
    uint4 *dst = reinterpret_cast<uint4 *>(L.ram + b * 64);
    dst[0] = src[0]; dst[1] = src[1]; dst[2] = src[2]; dst[3] = src[3];
    L.dirty |= 1ull << b;
  }
  L.ram[a] = (uint8_t)v;
}

__device__ __forceinline__ void power_on(Smem &sm, Lane &L, int tid) {
#pragma unroll
  for (int k = 0; k < 16; ++k) VREG(k) = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) sm.stk[k * kBlock + tid] = 0;
#pragma unroll
  for (int r = 0; r < 32; ++r) FBROW(r) = 0;
  L.pc = 0x200; L.I = 0; L.sp = 0; L.dt = 0; L.st = 0; L.halted = 0; L.keys = 0; L.draw = 0;
  L.dirty = 0;
  L.stk_dirty = 1;
}

// DXYN: XOR sprite rows into the framebuffer, VF = any lit pixel turned off.
__device__ __forceinline__ void draw(Smem &sm, Lane &L, int tid, uint32_t x, uint32_t y, uint32_t n,
                                     bool wrap) {
  uint32_t x0 = VREG(x) & 63u, y0 = VREG(y) & 31u, base = L.I & 0xFFFu;
  uint64_t hit = 0;
  for (uint32_t r = 0; r < n; ++r) {
    uint32_t yy = y0 + r;
    if (yy >= 32u) {
      if (!wrap) break;
      yy &= 31u;
    }
    uint32_t a = base + r;
    uint32_t byte = a <= 0xFFFu ? rd(sm, L, a) : 0u;
    uint64_t m = (uint64_t)byte << 56;
    m = wrap ? ((m >> x0) | (x0 ? (m << (64u - x0)) : 0ull)) : (m >> x0);
    uint64_t old = FBROW(yy);
    hit |= old & m;
    FBROW(yy) = old ^ m;
  }
  VREG(15) = hit ? 1u : 0u;
}

__device__ __forceinline__ void cycle(Smem &sm, Lane &L, const StepParams &p, int tid, uint32_t gid) {
  if (L.pc > 0xFFEu) { L.halted = 1; return; }
  uint32_t op = (rd(sm, L, L.pc) << 8) | rd(sm, L, L.pc + 1);
  L.pc = (L.pc + 2) & 0xFFFFu;
  uint32_t x = (op >> 8) & 15u, y = (op >> 4) & 15u, n = op & 15u, nn = op & 255u, nnn = op & 0xFFFu;
  switch (op >> 12) {
    case 0x0:
      if (op == 0x00E0u) {
#pragma unroll
        for (int r = 0; r < 32; ++r) FBROW(r) = 0;
      } else if (op == 0x00EEu) {
        if (L.sp == 0) { L.halted = 1; return; }
        L.sp--;
        L.pc = sm.stk[L.sp * kBlock + tid];
      }
      break;
    case 0x1: L.pc = nnn; break;
    case 0x2:
      if (L.sp == 16) { L.halted = 1; return; }
      sm.stk[L.sp * kBlock + tid] = (uint16_t)L.pc;
      L.sp++;
      L.stk_dirty = 1;
      L.pc = nnn;
      break;
    case 0x3: if (VREG(x) == nn) L.pc += 2; break;
    case 0x4: if (VREG(x) != nn) L.pc += 2; break;
    case 0x5:
      if (n) { L.halted = 1; return; }
      if (VREG(x) == VREG(y)) L.pc += 2;
      break;
    case 0x6: VREG(x) = nn; break;
    case 0x7: VREG(x) = (VREG(x) + nn) & 255u; break;
    case 0x8: {
      uint32_t a = VREG(x), b = VREG(y), r, f;
      bool vf_reset = (p.quirks & 16u) != 0;
      uint32_t s = (p.quirks & 1u) ? b : a;
      switch (n) {
        case 0x0: VREG(x) = b; return;
        case 0x1: VREG(x) = a | b; if (vf_reset) VREG(15) = 0; return;
        case 0x2: VREG(x) = a & b; if (vf_reset) VREG(15) = 0; return;
        case 0x3: VREG(x) = a ^ b; if (vf_reset) VREG(15) = 0; return;
        case 0x4: r = a + b; f = r >> 8; r &= 255u; break;
        case 0x5: r = (a - b) & 255u; f = a >= b; break;
        case 0x6: r = s >> 1; f = s & 1u; break;
        case 0x7: r = (b - a) & 255u; f = b >= a; break;
        case 0xE: r = (s << 1) & 255u; f = s >> 7; break;
        default: L.halted = 1; return;
      }
      VREG(x) = r;
      VREG(15) = f;  // flag written last (A15)
      break;
    }
    case 0x9:
      if (n) { L.halted = 1; return; }
      if (VREG(x) != VREG(y)) L.pc += 2;
      break;
    case 0xA: L.I = nnn; break;
    case 0xB: L.pc = (nnn + VREG((p.quirks & 4u) ? x : 0u)) & 0xFFFu; break;
    case 0xC: {
      uint32_t r = philox_out0(L.draw, L.episode, gid, 0u, (uint32_t)p.seed, (uint32_t)(p.seed >> 32));
      VREG(x) = r & nn & 255u;
      L.draw++;
      break;
    }
    case 0xD: draw(sm, L, tid, x, y, n, (p.quirks & 8u) != 0); break;
    case 0xE: {
      uint32_t down = (L.keys >> (VREG(x) & 15u)) & 1u;
      if (nn == 0x9Eu) { if (down) L.pc += 2; }
      else if (nn == 0xA1u) { if (!down) L.pc += 2; }
      else { L.halted = 1; return; }
      break;
    }
    default: {  // 0xF
      switch (nn) {
        case 0x07: VREG(x) = L.dt; break;
        case 0x0A:
          if (L.keys) VREG(x) = __ffs(L.keys) - 1;
          else L.pc -= 2;
          break;
        case 0x15: L.dt = VREG(x); break;
        case 0x18: L.st = VREG(x); break;
        case 0x1E: L.I = (L.I + VREG(x)) & 0xFFFFu; break;
        case 0x29: L.I = 0x50u + 5u * (VREG(x) & 15u); break;
        case 0x33: {
          uint32_t v = VREG(x);
          wr(sm, L, L.I & 0xFFFu, v / 100u);
          wr(sm, L, (L.I + 1u) & 0xFFFu, (v / 10u) % 10u);
          wr(sm, L, (L.I + 2u) & 0xFFFu, v % 10u);
          break;
        }
        case 0x55:
          for (uint32_t k = 0; k <= x; ++k) wr(sm, L, (L.I + k) & 0xFFFu, VREG(k));
          if (p.quirks & 2u) L.I = (L.I + x + 1u) & 0xFFFFu;
          break;
        case 0x65:
          for (uint32_t k = 0; k <= x; ++k) VREG(k) = rd(sm, L, (L.I + k) & 0xFFFu);
          if (p.quirks & 2u) L.I = (L.I + x + 1u) & 0xFFFFu;
          break;
        default: L.halted = 1; return;
      }
      break;
    }
  }
}

__device__ __forceinline__ void frame(Smem &sm, Lane &L, const StepParams &p, int tid, uint32_t gid) {
  for (uint32_t k = 0; k < p.ipf; ++k) {
    if (L.halted) break;
    cycle(sm, L, p, tid, gid);
  }
  if (!L.halted) {
    L.dt -= (L.dt != 0);
    L.st -= (L.st != 0);
  }
}

__device__ __forceinline__ uint32_t eval(const Program &P, Smem &sm, const Lane &L, int tid) {
  uint32_t tos = 0, sp = 0;
  for (uint32_t i = 0; i < P.len; ++i) {
    const ExprInsn in = P.ops[i];
    uint32_t a = 0, b = tos;
    if (in.op >= X_MUL) { --sp; a = sm.evs[sp * kBlock + tid]; }
    switch (in.op) {
      case X_CONST: case X_V: case X_I: case X_DT: case X_ST: {
        uint32_t v = in.op == X_CONST ? in.imm
                   : in.op == X_V   ? VREG(in.arg)
                   : in.op == X_I   ? L.I
                   : in.op == X_DT  ? L.dt : L.st;
        sm.evs[sp * kBlock + tid] = tos;
        ++sp;
        tos = v;
        break;
      }
      case X_MEM: tos = rd(sm, L, tos & 0xFFFu); break;
      case X_NEG: tos = 0u - tos; break;
      case X_NOT: tos = tos == 0u; break;
      case X_BNOT: tos = ~tos; break;
      case X_MUL: tos = a * b; break;
      case X_DIV: tos = b ? a / b : 0u; break;
      case X_MOD: tos = b ? a % b : 0u; break;
      case X_ADD: tos = a + b; break;
      case X_SUB: tos = a - b; break;
      case X_SHL: tos = b >= 32u ? 0u : a << b; break;
      case X_SHR: tos = b >= 32u ? 0u : a >> b; break;
      case X_LT: tos = a < b; break;
      case X_LE: tos = a <= b; break;
      case X_GT: tos = a > b; break;
      case X_GE: tos = a >= b; break;
      case X_EQ: tos = a == b; break;
      case X_NE: tos = a != b; break;
      case X_AND: tos = a & b; break;
      case X_XOR: tos = a ^ b; break;
      case X_OR: tos = a | b; break;
      case X_LAND: tos = (a != 0u) & (b != 0u); break;
      default: tos = (a != 0u) | (b != 0u); break;  // X_LOR
    }
  }
  return tos;
}

// ---------------------------------------------------------------- the step kernel
template <int MODE>
__global__ void __launch_bounds__(kBlock, 4)
octax_kernel(const __grid_constant__ StepParams p, const int32_t *__restrict__ actions,
             uint8_t *__restrict__ obs, float *__restrict__ reward, uint8_t *__restrict__ done_out,
             uint8_t *__restrict__ term_out, uint8_t *__restrict__ trunc_out) {
  extern __shared__ __align__(128) unsigned char smraw[];
  Smem &sm = *reinterpret_cast<Smem *>(smraw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t block0 = (uint64_t)blockIdx.x * kBlock;
  const uint64_t env = block0 + tid;
  const bool active = env < p.n;
  const uint64_t wbase = block0 + (uint64_t)warp * 32;
  const uint32_t h = p.head;
  uint64_t *__restrict__ ring = p.s.ring;
  uint64_t *__restrict__ obs64 = reinterpret_cast<uint64_t *>(obs);

  if (tid == 0) image_load_issue(sm, p.s.image);

  // ---- warp-cooperative prologue: obs planes 0..2 <- ring, framebuffer <- ring[h]
  if (MODE == MODE_STEP) {
    const uint32_t s0 = (h + 2) & 3, s1 = (h + 3) & 3, s2 = h & 3;
    const int ne = p.n > wbase ? (int)((p.n - wbase) < 32 ? (p.n - wbase) : 32) : 0;
#pragma unroll 4
    for (int e = 0; e < ne; ++e) {
      const uint64_t *rg = ring + (wbase + e) * 128;
      uint64_t r0 = rg[s0 * 32 + lane], r1 = rg[s1 * 32 + lane], r2 = rg[s2 * 32 + lane];
      uint64_t *ob = obs64 + (wbase + e) * 128;
      ob[lane] = r0;
      ob[32 + lane] = r1;
      ob[64 + lane] = r2;
      sm.fb[(warp * 32 + e) * kFbStride + lane] = bswap64(r2);
    }
  }

  Lane L;
  uint32_t steps = 0, prev = 0;
  int32_t ep_ret = 0;
  const uint32_t gid = (uint32_t)(p.env_offset + env);
  if (active) {
    uint4 v = p.s.regs[env];
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 16; ++k) VREG(k) = (w[k >> 2] >> (8 * (k & 3))) & 255u;
    uint4 c = p.s.ctrl[env];
    L.pc = c.x & 0xFFFFu; L.I = c.x >> 16;
    L.sp = c.y & 255u; L.dt = (c.y >> 8) & 255u; L.st = (c.y >> 16) & 255u; L.halted = c.y >> 24;
    L.draw = c.z; L.episode = c.w;
    uint4 b = p.s.book[env];
    steps = b.x; prev = b.y; ep_ret = (int32_t)b.z;
    uint4 s0 = p.s.stack[env * 2], s1 = p.s.stack[env * 2 + 1];
    uint32_t sw[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
#pragma unroll
    for (int k = 0; k < 16; ++k) sm.stk[k * kBlock + tid] = (uint16_t)(sw[k >> 1] >> (16 * (k & 1)));
    L.dirty = p.s.dirty[env];
    L.ram = p.s.ram + env * 4096ull;
    L.keys = 0;
    L.stk_dirty = 0;
  }
  __syncthreads();  // mbarrier init visible
  image_load_wait(sm);

  uint32_t did_reset = 0, err = 0, done = 0, term = 0, trunc = 0, finished = 0;
  float rew = 0.f;
  long long ret_acc = 0;
  if (active) {
    uint32_t frames_left, seg = 0;
    bool resetting;
    if (MODE == MODE_STEP) {
      int32_t a = actions[env];
      if (a < 0 || (uint32_t)a >= p.n_actions) { err = 1; a = 0; }
      L.keys = p.keymask[a];
      frames_left = p.frame_skip;
      resetting = false;
    } else {
      L.episode = 0;
      power_on(sm, L, tid);
      frames_left = 0;
      resetting = true;
    }
    for (;;) {
      for (; frames_left; --frames_left) frame(sm, L, p, tid, gid);
      if (!resetting) {
        uint32_t s = eval(p.score, sm, L, tid);
        int32_t d = (int32_t)(s - prev);
        rew = (float)d;
        prev = s;
        ep_ret = (int32_t)((uint32_t)ep_ret + (uint32_t)d);
        steps++;
        term = (eval(p.term, sm, L, tid) != 0u) || L.halted;
        trunc = p.max_steps && steps >= p.max_steps;
        done = term | trunc;
        if (!done) break;
        ret_acc = ep_ret;
        finished = 1;
        L.episode++;
        power_on(sm, L, tid);
        resetting = true;
        did_reset = 1;
      }
      if (seg < p.n_startup) {
        L.keys = p.startup_keys[seg];
        frames_left = p.startup_frames[seg];
        ++seg;
        continue;
      }
      L.keys = 0;
      steps = 0;
      prev = eval(p.score, sm, L, tid);
      ep_ret = 0;
      did_reset = 1;
      break;
    }
    if (MODE == MODE_STEP) {
      reward[env] = rew;
      done_out[env] = (uint8_t)done;
      if (term_out) term_out[env] = (uint8_t)term;
      if (trunc_out) trunc_out[env] = (uint8_t)trunc;
    }
  }
  __syncwarp();

  // ---- warp-cooperative epilogue: new ring slot + obs plane 3 (all planes on reset)
  {
    const uint32_t reset_mask = __ballot_sync(0xffffffffu, did_reset);
    const uint32_t sn = (h + 1) & 3;
    const int ne = p.n > wbase ? (int)((p.n - wbase) < 32 ? (p.n - wbase) : 32) : 0;
    for (int e = 0; e < ne; ++e) {
      uint64_t v = bswap64(sm.fb[(warp * 32 + e) * kFbStride + lane]);
      uint64_t *rg = ring + (wbase + e) * 128;
      uint64_t *ob = obs64 ? obs64 + (wbase + e) * 128 : nullptr;
      if (MODE == MODE_STEP) {
        rg[sn * 32 + lane] = v;
        ob[96 + lane] = v;
        if ((reset_mask >> e) & 1u) {
          rg[((h + 2) & 3) * 32 + lane] = v;
          rg[((h + 3) & 3) * 32 + lane] = v;
          rg[(h & 3) * 32 + lane] = v;
          ob[lane] = v; ob[32 + lane] = v; ob[64 + lane] = v;
        }
      } else {
        rg[lane] = v; rg[32 + lane] = v; rg[64 + lane] = v; rg[96 + lane] = v;
        if (ob) { ob[lane] = v; ob[32 + lane] = v; ob[64 + lane] = v; ob[96 + lane] = v; }
      }
    }
  }

  // ---- store lane state
  if (active) {
    uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < 16; ++k) w[k >> 2] |= (VREG(k) & 255u) << (8 * (k & 3));
    p.s.regs[env] = make_uint4(w[0], w[1], w[2], w[3]);
    p.s.ctrl[env] = make_uint4(L.pc | (L.I << 16), L.sp | (L.dt << 8) | (L.st << 16) | (L.halted << 24),
                               L.draw, L.episode);
    p.s.book[env] = make_uint4(steps, prev, (uint32_t)ep_ret, 0u);
    if (L.stk_dirty) {
      uint32_t sw[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        sw[k] = (uint32_t)sm.stk[(2 * k) * kBlock + tid] | ((uint32_t)sm.stk[(2 * k + 1) * kBlock + tid] << 16);
      p.s.stack[env * 2] = make_uint4(sw[0], sw[1], sw[2], sw[3]);
      p.s.stack[env * 2 + 1] = make_uint4(sw[4], sw[5], sw[6], sw[7]);
    }
    p.s.dirty[env] = L.dirty;
  }

  // ---- integer episode statistics (a12): warp reduce, CTA reduce, 4 atomics per CTA
  if (MODE == MODE_STEP) {
    unsigned long long r = (unsigned long long)ret_acc, f = finished, st = active ? 1u : 0u, er = err;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      r += __shfl_xor_sync(0xffffffffu, r, o);
      f += __shfl_xor_sync(0xffffffffu, f, o);
      st += __shfl_xor_sync(0xffffffffu, st, o);
      er |= __shfl_xor_sync(0xffffffffu, er, o);
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

// packed [n][4][32][8] -> bool [n][4][64][32]; one thread writes 16 bytes (16 y's of one x)
__global__ void expand_obs_kernel(uint64_t n, const uint8_t *__restrict__ packed, uint8_t *__restrict__ dense) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;  // unit of 16 output bytes
  uint64_t total = n * 4 * 64 * 2;
  if (i >= total) return;
  uint32_t yh = i & 1, x = (i >> 1) & 63;
  uint64_t plane = i >> 7;  // env*4 + p
  const uint8_t *src = packed + plane * 256;
  uint32_t w[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t y = yh * 16 + q * 4 + k;
      acc |= ((uint32_t)(src[y * 8 + (x >> 3)] >> (7 - (x & 7))) & 1u) << (8 * k);
    }
    w[q] = acc;
  }
  reinterpret_cast<uint4 *>(dense)[i] = make_uint4(w[0], w[1], w[2], w[3]);
}

// canonical per-env state (DESIGN.md layout), one CTA of 128 threads per requested env
__global__ void get_states_kernel(StepParams p, const uint64_t *__restrict__ ids, uint8_t *__restrict__ out) {
  const uint64_t env = ids[blockIdx.x];
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
  const uint8_t *rg = reinterpret_cast<const uint8_t *>(p.s.ring + env * 128);
  for (int i = t; i < 256; i += blockDim.x) {
    c[80 + i] = rg[(h & 3) * 256 + i];
    c[336 + i] = rg[((h + 1) & 3) * 256 + i];
    c[592 + i] = rg[((h + 2) & 3) * 256 + i];
    c[848 + i] = rg[((h + 3) & 3) * 256 + i];
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
  uint8_t *rg = reinterpret_cast<uint8_t *>(p.s.ring + env * 128);
  for (int i = t; i < 256; i += blockDim.x) {
    rg[(h & 3) * 256 + i] = c[80 + i];
    rg[((h + 1) & 3) * 256 + i] = c[336 + i];
    rg[((h + 2) & 3) * 256 + i] = c[592 + i];
    rg[((h + 3) & 3) * 256 + i] = c[848 + i];
  }
  uint8_t *ram = p.s.ram + env * 4096ull;
  for (int i = t; i < 4096; i += blockDim.x) ram[i] = c[1104 + i];
}

// ---------------------------------------------------------------- launchers
static bool g_attr_set[2] = {false, false};

cudaError_t launch_step(const StepParams &p, int mode, const int32_t *actions, uint8_t *obs, float *reward,
                        uint8_t *done, uint8_t *term, uint8_t *trunc, cudaStream_t stream) {
  const size_t smem = sizeof(Smem);
  const unsigned grid = (unsigned)((p.n + kBlock - 1) / kBlock);
  if (mode == MODE_STEP) {
    if (!g_attr_set[0]) {
      cudaError_t e = cudaFuncSetAttribute(octax_kernel<MODE_STEP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
      if (e != cudaSuccess) return e;
      g_attr_set[0] = true;
    }
    octax_kernel<MODE_STEP><<<grid, kBlock, smem, stream>>>(p, actions, obs, reward, done, term, trunc);
  } else {
    if (!g_attr_set[1]) {
      cudaError_t e = cudaFuncSetAttribute(octax_kernel<MODE_RESET>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
      if (e != cudaSuccess) return e;
      g_attr_set[1] = true;
    }
    octax_kernel<MODE_RESET><<<grid, kBlock, smem, stream>>>(p, nullptr, obs, nullptr, nullptr, nullptr, nullptr);
  }
  return cudaGetLastError();
}

cudaError_t launch_gen_actions(uint64_t n, uint64_t env_offset, uint64_t aseed, uint64_t t, uint32_t n_actions,
                               int32_t *out, cudaStream_t stream) {
  const unsigned grid = (unsigned)((n + 255) / 256);
  gen_actions_kernel<<<grid, 256, 0, stream>>>(n, env_offset, aseed, t, n_actions, out);
  return cudaGetLastError();
}

cudaError_t launch_expand_obs(uint64_t n, const uint8_t *packed, uint8_t *dense, cudaStream_t stream) {
  uint64_t total = n * 4 * 64 * 2;
  const unsigned grid = (unsigned)((total + 255) / 256);
  expand_obs_kernel<<<grid, 256, 0, stream>>>(n, packed, dense);
  return cudaGetLastError();
}

cudaError_t launch_get_states(const StepParams &p, const uint64_t *ids, uint64_t count, uint8_t *out,
                              cudaStream_t stream) {
  get_states_kernel<<<(unsigned)count, 128, 0, stream>>>(p, ids, out);
  return cudaGetLastError();
}

cudaError_t launch_set_state(const StepParams &p, uint64_t env, const uint8_t *canon, cudaStream_t stream) {
  set_state_kernel<<<1, 128, 0, stream>>>(p, env, canon);
  return cudaGetLastError();
}

}  // namespace octax
