// octax_dev.cuh -- internal (non-ABI) structures shared by the host library and
// the sm_100a kernels of the B200 Octax step.  Nothing here is shared with oracle/.
#pragma once
#include <cstdint>

namespace octax {

#ifndef OCTAX_BLOCK
#define OCTAX_BLOCK 128
#endif
#ifndef OCTAX_MINB
#define OCTAX_MINB 5
#endif
constexpr int kBlock = OCTAX_BLOCK;  // envs (threads) per CTA (a multiple of 32)
constexpr int kMinBlocks = OCTAX_MINB;  // resident CTAs per SM the step kernel is built for
constexpr int kMaxStartup = 32;
#ifndef OCTAX_HOST_CHUNKS
#define OCTAX_HOST_CHUNKS 8
#endif
constexpr uint32_t kMaxHostChunks = OCTAX_HOST_CHUNKS;  // pipelined host steps: launches per step (octax_api.cpp host_step)
constexpr int kMaxOps = 64;
constexpr int kMaxDepth = 8;
constexpr uint32_t kImageBytes = 4096;
constexpr uint32_t kWordEntries = 65536;  // warp kernel word table: one entry per 16-bit PC
constexpr uint32_t kDescEntries = 256;
constexpr uint32_t kStageBytes = kImageBytes + 4 * kDescEntries;  // image + decode table, one bulk copy

// Per-handle decode table (quirks folded in), indexed by desc_index(op): one
// 32-bit descriptor of what the instruction does, so the warp-uniform core tests
// descriptor bits instead of re-deriving the class from the opcode every cycle.
// E/F entries carry the expected y nibble (bits 28..31, checked under D_YCHK): with
// the injective nibble hash below, (hi, hash, y) determines the whole word.
enum : uint32_t {
  // skips: D_SKIP = conditional skip; the condition is VX == (D_BVY ? VY : NN), or with
  // D_SKEY "key VX & 15 is down"; D_SINV negates it (4XNN, 9XY0, EXA1)
  D_OK = 1u << 0, D_YCHK = 1u << 1, D_SKIP = 1u << 2, D_SINV = 1u << 3, D_BVY = 1u << 4,
  D_SKEY = 1u << 5, D_RARE = 1u << 6, D_WVX = 1u << 7, D_WVF = 1u << 8, D_VSADD = 1u << 9,
  D_VSALU = 1u << 10, D_VSDT = 1u << 11, D_WAIT = 1u << 12, D_PCJ = 1u << 13, D_CALL = 1u << 14,
  D_BJMP = 1u << 15, D_INNN = 1u << 16, D_IADD = 1u << 17, D_IFONT = 1u << 18, D_DTW = 1u << 19,
  D_STW = 1u << 20, D_RND = 1u << 21, D_MEM = 1u << 22, D_DRAW = 1u << 23,
  // predecoded-entry only (never in the descriptor table): the skip truth table (bit
  // 1 + i = skip when i = [VX == operand] | [key VX down] << 1), VY-operand flag, faults
  E_SKL = 0xFu << 1, E_BVY = 1u << 5, E_BAD = 1u << 25, E_RET = 1u << 26, E_CLS = 1u << 27,
  D_EXEC = 0x00FFFFC0u  // descriptor bits that carry over into an entry unchanged
};

// hi << 4 | low nibble; for EXnn / FXnn the nibble is (n - 2y) & 15, which is
// injective on the 11 defined E/F low bytes (9E A1 | 07 0A 15 18 1E 29 33 55 65).
#ifdef __CUDACC__
__host__ __device__
#endif
inline uint32_t desc_index(uint32_t op) {
  const uint32_t hi = op >> 12, y = (op >> 4) & 15u, n = op & 15u;
  return (hi << 4) | (hi >= 14u ? ((n + 14u * y) & 15u) : n);
}

// Predecoded instruction: what the core needs from the 16-bit word at a PC, with every
// decision that depends on the word alone taken once (per handle, on the host, for all
// 4096 PCs of the pristine image; on the device only for a PC in a dirty RAM block).
//   .x = execution flags: D_* bits of D_EXEC, E_SKL / E_BVY (skips), E_BAD / E_RET / E_CLS
//   .y = kx | ky << 9 | (sp delta + 1) << 18 | nnn << 20 (nn at bits 20..27, x 28..31), with
//        k* = (k >> 2) << 7 | (k & 3) for register index k (its smem V offset within the
//        lane's bank, see VREG) -- kx addresses the register the word reads as "VX":
//        V[x], or V0 for BNNN without the JUMP_VX quirk; sp delta = +1 for 2NNN, -1 for
//        00EE (a new SP outside 0..16 is a stack fault).
//   D_RARE marks the vote-gated classes (00E0, CXNN, FX33/55/65).
//   8XYn (D_VSALU): .y bits 24..31 (the x / high-nn fields, which the core does not read
//   for 8XYn) hold the ALU operation one-hot (A_*), so the core selects the result with
//   single-bit tests instead of comparing n; for 8XYE without the SHIFT_VY quirk the VY
//   offset is VX's, so VX << 1 is the A_ADD of VX and VX.
enum : uint32_t {
  A_OR = 1u << 24, A_AND = 1u << 25, A_XOR = 1u << 26, A_ADD = 1u << 27,  // A_ADD: 8XY4, 8XYE
  A_SUB = 1u << 28, A_RSUB = 1u << 29, A_SHR = 1u << 30,                   // 8XY5, 8XY7, 8XY6
  A_SRCY = 1u << 31  // SHIFT_VY quirk: 8XY6 / 8XYE shift VY (never set for the modern profile)
};
// every 16-bit PC (entries past 0xFFE halt, A17, so no clamp), plus a second 64K of E_BAD
// entries fetched by lanes that are halted on entry or past n (PC bit 16 set in the kernel)
constexpr uint32_t kDecEntries = 131072;
#ifdef __CUDACC__
__host__ __device__
#endif
inline void make_entry(uint32_t op, const uint32_t *dtab, uint32_t quirks, uint32_t &ex, uint32_t &ey) {
  const uint32_t x = (op >> 8) & 15u, y = (op >> 4) & 15u, nn = op & 255u;
  const uint32_t d = dtab[desc_index(op)];
  const bool bad = (d & D_OK) == 0u || ((d & D_YCHK) != 0u && y != (d >> 28));
  uint32_t f = bad ? E_BAD : (d & D_EXEC);
  if (!bad && (d & D_SKIP) != 0u) {
    const uint32_t lut = (d & D_SKEY) ? 0xCu : 0xAu;  // skip when the key is down / VX == operand
    f |= ((d & D_SINV) ? (~lut & 0xFu) : lut) << 1;
    if (d & D_BVY) f |= E_BVY;
  }
  if (op == 0x00EEu) f |= E_RET;
  if (op == 0x00E0u) f |= E_CLS;
  if ((f & (E_CLS | D_RND | D_MEM)) != 0u) f |= D_RARE;
  const uint32_t dsp = (f & E_RET) ? 0u : (f & D_CALL) ? 2u : 1u;
  const uint32_t rx = ((d & D_BJMP) != 0u && (quirks & 4u) == 0u) ? 0u : x;  // 4 = OCTAX_Q_JUMP_VX
  ex = f;
  const uint32_t kx = ((rx >> 2) << 7) | (rx & 3u);
  const uint32_t n = op & 15u, shy = quirks & 1u;  // 1 = OCTAX_Q_SHIFT_VY
  const uint32_t ry = ((f & D_VSALU) != 0u && n == 0xEu && !shy) ? x : y;  // 8XYE: VX + VX
  const uint32_t ky = ((ry >> 2) << 7) | (ry & 3u);
  ey = kx | (ky << 9) | (dsp << 18) | (nn << 20) | (x << 28);
  if ((f & D_VSALU) != 0u) {
    const uint32_t a = n == 1u ? A_OR : n == 2u ? A_AND : n == 3u ? A_XOR : n == 4u ? A_ADD
                     : n == 5u ? A_SUB : n == 7u ? A_RSUB : n == 6u ? (A_SHR | (shy ? A_SRCY : 0u))
                     : n == 0xEu ? (A_ADD | (shy ? A_SRCY : 0u)) : 0u;  // n == 0: VX = VY
    ey = (ey & 0x00FFFFFFu) | a;
  }
}

// expression bytecode (postfix, evaluated with top-of-stack in a register)
enum ExprOp : uint8_t {
  X_CONST = 0, X_V, X_I, X_DT, X_ST,
  X_VDIV, X_VMOD,  // push V[arg] / c, V[arg] % c for a constant c = pad (fused at create from
                   // "V[n] c /" and "V[n] c %"): q = (V * imm) >> 16, imm = 2^16 / c + 1, exact for
                   // the byte V when c <= 255; imm = 0 for c > 255 (q = 0)
  X_MEM, X_NEG, X_NOT, X_BNOT,
  X_MUL, X_DIV, X_MOD, X_ADD, X_SUB, X_SHL, X_SHR,
  X_LT, X_LE, X_GT, X_GE, X_EQ, X_NE, X_AND, X_XOR, X_OR, X_LAND, X_LOR
};

struct ExprInsn {
  uint8_t op;
  uint8_t arg;
  uint16_t pad;
  uint32_t imm;
};

struct Program {
  ExprInsn ops[kMaxOps];
  uint32_t len;
  uint32_t depth;
  // the program's shape when it is one of the common one- to three-op forms, evaluated without
  // the bytecode loop: 0 = general, 1 = constant ka, 2 = V[ka], 3 = V[ka] == kb, 4 = V[ka] != kb
  uint32_t kind;
  uint32_t ka, kb;
};

// Device-resident per-env state, structure-of-arrays (one entry per local env).
struct DevState {
  uint4 *regs;       // [n]    V0..VF, byte k of the 16 = Vk
  uint4 *ctrl;       // [n]    {PC | I<<16, SP | DT<<8 | ST<<16 | halted<<24, draw, episode}
  uint4 *book;       // [n]    {steps, prev_score, ep_ret, 0}
  uint4 *stack;      // [n*2]  16 x u16 return addresses
  uint64_t *dirty;   // [n]    copy-on-write block mask (64 blocks of 64 B)
  uint8_t *ram;      // [n*4096] RAM backing; only dirty blocks are valid
  uint64_t *ring;    // [4][n_pad][32] display history, slot-major (n_pad = n rounded up to
                     // kBlock, so a CTA's 128 envs are one contiguous 32 KB block per slot);
                     // u64 = one row in packed byte order; position j of env e holds row
                     // j ^ (e & 14) -- the shared-memory framebuffer's swizzle (kSwz), so ring <->
                     // smem moves are plain TMA bulk copies
  uint64_t ring_stride;  // u64 per ring slot = n_pad * 32
  unsigned long long *stats;  // [4] {returns, episodes, steps, err}
  const uint8_t *image;       // [4096] pristine image: zeros, font at 0x50, ROM at 0x200
  const uint2 *dec;           // [kDecEntries] predecoded instruction at every PC (make_entry)
  const uint16_t *words;      // [4096] the pristine image's 16-bit word at every PC <= 0xFFE
                              // (warp-per-env kernel fetch: one load, no byte assembly)
};

struct StepParams {
  DevState s;
  // optional per-step extra outputs (octax_step_ex), nullptr when not requested
  uint8_t *final_obs;      // packed [n][4][32][8]: obs of the terminal transition, done envs only
  uint8_t *frame_out;      // packed [n][32][8]: this step's newest display (obs plane 3), all envs
  int32_t *ep_ret_out;     // return of the episode that ended this step (0 if none)
  uint32_t *ep_len_out;    // its length in steps (0 if none)
  uint32_t *reset_count;   // deferred resets (specs with startup segments): [1] counter and
  uint32_t *reset_ids;     // [n] env ids appended by the step kernel, run by reset_kernel
  uint64_t n;
  uint64_t env_offset;
  uint32_t block_base;    // first CTA block of this launch (a chunk of the envs, host paths)
  uint32_t block_count;   // CTA blocks in this launch; 0 = all blocks from block_base
  uint64_t seed;
  uint32_t head;          // ring slot holding the current display
  uint32_t frame_skip;
  uint32_t ipf;
  uint32_t max_steps;
  uint32_t quirks;
  uint32_t obs_format;
  uint32_t stack_frames;  // OCTAX_OBS_STACK_FRAMES: obs = last 4 frames of the step
  uint32_t n_actions;     // n_action_keys + 1
  uint32_t n_startup;
  uint32_t warp;          // 1: the warp-per-env kernel runs this launch (octax_set_kernel), 0: lane-per-env
  // fused rollout (MODE_ROLLOUT, octax_rollout): T steps per launch; step t's obs at obs + t *
  // obs_stride (u64 units), reward / done / terminated / truncated at [t * out_stride + env];
  // actions [T][n] if given, else generated in-kernel for step index t0 + t with key aseed
  uint32_t T;
  uint64_t aseed;
  uint64_t t0;
  uint64_t obs_stride;
  uint64_t out_stride;
  uint16_t keymask[17];   // action -> key mask
  uint16_t pad0;
  uint32_t startup_keys[kMaxStartup];
  uint32_t startup_frames[kMaxStartup];
  Program score;
  Program term;
};

enum Mode : int { MODE_STEP = 0, MODE_RESET = 1, MODE_ROLLOUT = 2, MODE_ROLLOUT_NOOBS = 3 /* kernel only */ };

}  // namespace octax
