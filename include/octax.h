/*
 * octax.h -- C ABI of the B200-native batched Octax environment step.
 *
 * The operation: the batched RL environment step of Octax (arXiv 2510.01764),
 * i.e. for each of n independent CHIP-8 virtual machines
 *   1. map the discrete action to a key mask, held for the whole step
 *      ("Actions map from discrete RL outputs to game-specific key subsets
 *      plus a no-op option"; P:156 action_set; reading A5: action 0 = no-op),
 *   2. run frame_skip frames ("each step represents 4 frames"), each frame
 *      = instructions_per_frame fetch/decode/execute cycles of the 35-opcode
 *      CHIP-8 ISA (§3.2, App. A.3) followed by the 60 Hz
 *      delay/sound timer decrement, with DXYN drawing sprites by XOR onto
 *      the 64x32 1-bit display and setting VF on collision,
 *   3. evaluate the game's score and termination expressions over registers and
 *      memory (§3.3; App. D) -> reward = signed score
 *      delta (A6/A7), terminated = expr != 0 or VM fault (A17), truncated =
 *      steps >= max_episode_steps (A9),
 *   4. emit the 4-frame stacked observation ("(4, 64, 32) boolean arrays";
 *      A3: the last four step-end displays, oldest first),
 *   5. auto-reset finished envs in the same step, running the startup segments
 *      (P:146, P:158 startup_instructions; A10 Gymnax convention: the returned
 *      obs is the reset obs; reward/done come from the terminal transition).
 *      This deviates from SPEC S:409's "final observation, then reset before the
 *      next step": the terminal obs SPEC would return is available as
 *      octax_step_ex's final_obs_out (written for done envs).
 * Readings A1..A33 are listed in DESIGN.md.  Two interchangeable step kernels run the
 * step (octax_set_kernel below): one thread per env, or one warp per env for small batches.
 *
 * Memory: the library owns all VM state (device memory of the handle's device).
 * Buffers passed to octax_step / octax_reset / octax_gen_actions / octax_stats_device
 * are CALLER-OWNED DEVICE buffers, contiguous, used stream-ordered on the
 * handle's stream; those calls never synchronise the host.  Buffers passed to
 * octax_step_host, octax_stats, octax_get_state(s) and octax_set_state are host
 * buffers; those calls synchronise the handle's stream.
 * Step / rollout / reset kernels are launched with programmatic stream serialization (PDL):
 * the next launch's CTAs may be scheduled while the previous kernel on the stream drains, but
 * each waits for that kernel to complete and its writes to be visible before touching any
 * buffer, so the observable order is plain stream order.
 *
 * Layouts (per env j, local index 0..n-1):
 *   actions  int32  [n]
 *   obs      OCTAX_OBS_PACKED:      uint8 [n][4][32][8]  plane p (0 = oldest), row y,
 *                                    byte b = pixels 8b..8b+7, MSB = leftmost
 *            OCTAX_OBS_BOOL_XMAJOR: uint8 0/1 [n][4][64][32] = [frame][x][y]
 *   reward   float32 [n]   done / terminated / truncated  uint8 0/1 [n]
 *
 * Errors: every function returns octax_status; 0 = OK.  A message for the last
 * failing call on the calling thread is available from octax_last_error().
 * Device-side anomalies cannot fail a step: an out-of-range action is treated as
 * the no-op and sets a sticky flag reported by octax_stats (OCTAX_E_DEVICE);
 * VM faults (invalid opcode, stack over/underflow, PC past 0xFFE) halt the lane,
 * which reports terminated = 1 and is auto-reset (A17).
 *
 * Thread safety: one host thread at a time per handle; handles are independent.
 */
#ifndef OCTAX_H
#define OCTAX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OCTAX_ABI_VERSION 1u

typedef enum {
  OCTAX_OK = 0,
  OCTAX_E_INVALID_ARG = -1,  /* NULL pointer, n_envs = 0, env index out of range ... */
  OCTAX_E_ROM_EMPTY = -2,    /* rom_len == 0                                         */
  OCTAX_E_ROM_TOO_LARGE = -3,/* rom_len > 3584 = 4096 - 0x200          */
  OCTAX_E_SPEC = -4,         /* bad spec field, e.g. duplicate / >15 action key      */
  OCTAX_E_EXPR = -5,         /* expression syntax error; byte offset in the message  */
  OCTAX_E_CUDA = -6,         /* CUDA runtime error (message carries cudaGetErrorString) */
  OCTAX_E_OOM = -7,          /* device or host allocation failed                     */
  OCTAX_E_DEVICE = -8        /* sticky device flag: an out-of-range action was seen  */
} octax_status;

/* quirk bits; 0 = "modern" profile (A14) */
enum {
  OCTAX_Q_SHIFT_VY = 1,         /* 8XY6/8XYE shift VY into VX                 */
  OCTAX_Q_LOADSTORE_INC_I = 2,  /* FX55/FX65 leave I = I + X + 1              */
  OCTAX_Q_JUMP_VX = 4,          /* BNNN adds VX instead of V0                 */
  OCTAX_Q_WRAP_SPRITES = 8,     /* DXYN wraps at the edges instead of clipping */
  OCTAX_Q_VF_RESET = 16         /* 8XY1/2/3 clear VF                          */
};

enum { OCTAX_OBS_PACKED = 0, OCTAX_OBS_BOOL_XMAJOR = 1,
       /* flag, OR-ed with a layout: stack the displays after the last 4 FRAMES of the step
          (the other reading of P:146 "4-frame stacking") instead of the last
          4 step-end displays (A3, default); with frame_skip < 4 the missing leading planes
          repeat the step-start display; reset obs = 4 copies of the reset display */
       OCTAX_OBS_STACK_FRAMES = 16 };

#define OCTAX_MAX_STARTUP 32u   /* startup segments per spec                   */
#define OCTAX_MAX_EXPR_OPS 64u  /* compiled expression length (ops)            */
#define OCTAX_MAX_EXPR_DEPTH 8u /* evaluation stack depth                      */
#define OCTAX_CANON_BYTES 5200u /* canonical per-env state, layout in DESIGN.md */

/* Startup segment (A11): hold `keymask` for `frames` frames at reset. */
typedef struct {
  uint16_t keymask;
  uint32_t frames;
} octax_startup_seg;

/* Per-game environment definition (P:1568-1608 game module format).
 * All strings and arrays are COPIED by octax_create. */
typedef struct {
  uint32_t abi_version;              /* must be OCTAX_ABI_VERSION                   */
  const char *score_expr;            /* e.g. "V5", "(V14 // 10) - (V14 % 10)"        */
  const char *terminated_expr;       /* e.g. "V14 == 0", "(V9 == 0) | (V12 >= 0x3E)" */
  const uint8_t *action_keys;        /* 1..16 distinct keys 0..15; action a>=1 holds
                                        key action_keys[a-1]; action 0 = no-op       */
  uint32_t n_action_keys;
  const octax_startup_seg *startup;  /* may be NULL when n_startup == 0              */
  uint32_t n_startup;                /* <= OCTAX_MAX_STARTUP                         */
  uint32_t frame_skip;               /* >= 1, default 4                      */
  uint32_t instructions_per_frame;   /* >= 1, default 12 (A1)                        */
  uint32_t max_episode_steps;        /* 0 = no truncation, default 10000 (A9)        */
  uint32_t quirks;                   /* OCTAX_Q_* bits                               */
  uint32_t obs_format;               /* OCTAX_OBS_PACKED | OCTAX_OBS_BOOL_XMAJOR, optionally
                                        | OCTAX_OBS_STACK_FRAMES                     */
} octax_game_spec;

/* Device placement.  env_offset / total_envs: this handle simulates global env
 * ids env_offset .. env_offset+n_envs-1 (multi-GPU sharding, A13: every random
 * draw is keyed by the GLOBAL id, so trajectories do not depend on sharding).
 * cuda_stream is a cudaStream_t (NULL = legacy default stream). */
typedef struct {
  int device;
  void *cuda_stream;
  uint64_t env_offset;
  uint64_t total_envs; /* informational; 0 = n_envs */
} octax_device_opts;

typedef struct octax_env octax_env;

/* Validate rom/spec, compile the expressions, allocate ~5.2 KB of device state
 * per env, and run the episode-0 reset of every env (as octax_reset(seed, NULL)).
 * opts may be NULL (device 0, default stream, offset 0). */
octax_status octax_create(const uint8_t *rom, size_t rom_len, const octax_game_spec *spec,
                          uint64_t n_envs, uint64_t seed, const octax_device_opts *opts,
                          octax_env **out);

/* Reset every env: batch seed := seed, episode := 0, power-on + startup.
 * Clears the statistics.  obs_out (device, may be NULL) receives the reset obs. */
octax_status octax_reset(octax_env *e, uint64_t seed, void *obs_out);

/* One environment step for all n envs (one kernel launch, stream-ordered).
 * actions, obs_out, reward_out, done_out: device buffers (required);
 * terminated_out / truncated_out: device buffers or NULL. */
octax_status octax_step(octax_env *e, const int32_t *actions, void *obs_out, float *reward_out,
                        uint8_t *done_out, uint8_t *terminated_out, uint8_t *truncated_out);

/* Optional extra outputs of octax_step_ex (all DEVICE buffers, each may be NULL):
 *  final_obs_out       obs of the TERMINAL transition (the 4 stacked displays before the
 *                      same-step auto-reset, A10), same layout as obs_out; written for envs
 *                      with done = 1 only, other rows untouched.  With it a caller gets
 *                      SPEC's final-observation convention on top of Gymnax's.
 *  episode_return_out  int32 [n]: return (sum of rewards) of the episode that ended this
 *                      step, 0 where done = 0 (S:417 telescoping).
 *  episode_length_out  uint32 [n]: its length in steps, 0 where done = 0. */
typedef struct {
  void *final_obs_out;
  int32_t *episode_return_out;
  uint32_t *episode_length_out;
  void *frame_out;      /* uint8 [n][32][8] packed: this step's newest display (obs plane 3) alone,
                           contiguous, all envs -- what a consumer keeping its own 3-display
                           history needs (octax_step_host_frame) */
} octax_step_extras;

/* octax_step plus the extras above (extras may be NULL = octax_step). */
octax_status octax_step_ex(octax_env *e, const int32_t *actions, void *obs_out, float *reward_out,
                           uint8_t *done_out, uint8_t *terminated_out, uint8_t *truncated_out,
                           const octax_step_extras *extras);

/* Same step with HOST buffers (pinned recommended): copies actions host->device, steps the envs
 * on internal device buffers, copies obs/reward/done back and synchronises.  terminated_out /
 * truncated_out may be NULL.  Large batches are stepped in several launches over consecutive
 * env blocks; each block's results are copied back on a second stream while the next block's
 * launch runs (the PCIe copy, not the kernel, bounds a host step).  Results are identical to
 * octax_step. */
octax_status octax_step_host(octax_env *e, const int32_t *actions_host, void *obs_host,
                             float *reward_host, uint8_t *done_host, uint8_t *terminated_host,
                             uint8_t *truncated_host);

/* Host step that ships only what changed (NEXT-3 host variant): like octax_step_host, but the
 * device->host copy carries the NEWEST display (uint8 [n][32][8] packed, = obs plane 3) instead of
 * the 4-plane stack -- 261 instead of 1,029 bytes per env.  The caller keeps the three previous
 * displays: obs = [d(t-3), d(t-2), d(t-1), frame], except that an env with done = 1 was reset in
 * this step (A10), so its 4 planes all equal the frame.  A host history started from octax_reset's
 * obs (4 equal planes) reproduces octax_step's obs exactly (tests/test_gpu_parity.py).  Valid for
 * the default stacking (A3); with OCTAX_OBS_STACK_FRAMES the frame is still the newest display but
 * the other planes are intermediate frames the host cannot rebuild.  Synchronises the stream. */
octax_status octax_step_host_frame(octax_env *e, const int32_t *actions_host, void *frame_host,
                                   float *reward_host, uint8_t *done_host, uint8_t *terminated_host,
                                   uint8_t *truncated_host);

/* Synthetic benchmark actions (device, int32 [n]):
 * a_j = Philox4x32-10(ctr = {t_lo, t_hi, gid_j, 1}, key = aseed).out0 mod n_actions. */
octax_status octax_gen_actions(octax_env *e, uint64_t aseed, uint64_t t, int32_t *actions_out);

/* Fused rollout (SURVEY 8(d) d.3 / d.8 mode "fused"; the paper's 100-step rollouts):
 * T consecutive environment steps of all n envs in ONE kernel launch, the VM state and the
 * framebuffer kept on chip across the T steps.  Bit-identical to T octax_step calls:
 *  - step t (0 <= t < T) takes actions[t*n + j] (DEVICE int32 [T][n]) when actions != NULL,
 *    else the action octax_gen_actions(aseed, t0 + t) would produce, generated in the kernel
 *    (Philox4x32-10, ctr = {t_lo, t_hi, gid, 1}, key = aseed; SURVEY 2.3 K6 fused into K1);
 *  - step t's obs goes to (uint8*)obs_out + t*obs_step_stride (bytes, a multiple of 16; 0 =
 *    every step overwrites the same [n] obs buffer, so the last step's obs remains), its
 *    reward / done / terminated / truncated to [t*out_step_stride + j] (elements; 0 = same
 *    buffers every step).  terminated_out / truncated_out may be NULL.  All DEVICE buffers.
 *  - obs_out may be NULL: no observation is written (rewards / dones only, e.g. policy-free
 *    evaluation); the display history is still kept, so later steps' obs are unaffected.
 *  - a non-zero stride must cover all n envs (obs: >= n * 1024 bytes; outputs: >= n).
 * Same-step auto-reset (A10) runs inline, also for specs with startup segments.  Either
 * stacking mode; either layout: with OCTAX_OBS_BOOL_XMAJOR the kernel writes packed obs to a
 * library staging buffer ([T][n] packed, or the last step's with stride 0) that
 * expand_obs_kernel expands into obs_out after it (obs_step_stride 0 or n * 8192).  T = 0 is a
 * no-op.  Stream-ordered, no host synchronisation; the statistics count all T steps. */
octax_status octax_rollout(octax_env *e, uint32_t T, const int32_t *actions, uint64_t aseed, uint64_t t0,
                           void *obs_out, uint64_t obs_step_stride, float *reward_out, uint8_t *done_out,
                           uint8_t *terminated_out, uint8_t *truncated_out, uint64_t out_step_stride);

/* Episode statistics since create/reset: {sum of returns of finished episodes,
 * finished episodes, env steps, error flags} (int64).  Synchronises the stream.
 * Returns OCTAX_E_DEVICE (after filling out4) when the sticky error flag is set. */
octax_status octax_stats(octax_env *e, int64_t out4[4]);

/* Same four int64 written stream-ordered to a DEVICE buffer (for NCCL reduction). */
octax_status octax_stats_device(octax_env *e, int64_t *out4_device);

/* Canonical per-env state (OCTAX_CANON_BYTES, host buffer), for tests/checkpoints.
 * octax_get_states gathers `count` envs (local indices) into canon_out[count][5200]. */
octax_status octax_get_state(octax_env *e, uint64_t env, uint8_t *canon_out);
octax_status octax_get_states(octax_env *e, const uint64_t *envs, uint64_t count,
                              uint8_t *canon_out);
octax_status octax_set_state(octax_env *e, uint64_t env, const uint8_t *canon_in);

/* Per-env 64-bit state digests: FNV-1a 64 (offset 0xCBF29CE484222325, prime 0x100000001B3)
 * over the 5,200 canonical bytes of octax_get_state, for local envs [first, first+count).
 * digests_out: host uint64 [count] or NULL; sum_out: host, the sum of the digests mod 2^64,
 * or NULL (not both NULL).  Because every trajectory is keyed by the global env id (A13), the
 * digests of an env are identical for any sharding.
 * Synchronises the stream; OCTAX_E_INVALID_ARG on a bad range. */
octax_status octax_state_digests(octax_env *e, uint64_t first, uint64_t count, uint64_t *digests_out,
                                 uint64_t *sum_out);

/* Which step kernel runs the handle's launches (every entry point above; results identical,
 * bit for bit -- both follow oracle/ c.1 and share the device state layout, so the choice may
 * change between any two calls):
 *   OCTAX_KERNEL_LANE -- one thread per env, 128 envs per CTA (the throughput kernel: the
 *     GPU-filling batches of configs 3-5, 1M envs per GPU);
 *   OCTAX_KERNEL_WARP -- one warp per env, the VM state in the warp's registers, no
 *     divergence (the paper's lockstep bottleneck): lower latency per step, for batches
 *     too small to fill the GPU with lane-per-env warps (512..8,192 envs);
 *   OCTAX_KERNEL_AUTO -- WARP when n <= OCTAX_WARP_AUTO_MAX_ENVS (the measured crossover;
 *     environment variable OCTAX_WARP_AUTO_MAX overrides it at create), else LANE.  The choice
 *     sees only this handle: several small handles stepped concurrently on one GPU that together
 *     exceed ~4,096 envs run faster with LANE on each (16 x 4,096 envs: 1.26e9 vs 2.9e8 env
 *     steps/s, bench.py `concurrent_handles`). 
 * octax_set_kernel: OCTAX_E_INVALID_ARG for another value.  octax_get_kernel: the kernel in
 * use (LANE or WARP), never AUTO. */
#define OCTAX_KERNEL_AUTO 0
#define OCTAX_KERNEL_LANE 1
#define OCTAX_KERNEL_WARP 2
#define OCTAX_WARP_AUTO_MAX_ENVS 4096
octax_status octax_set_kernel(octax_env *e, int kernel);
octax_status octax_get_kernel(octax_env *e, int *kernel_out);

/* Handle facts: n_envs, n_actions, obs bytes per env, device bytes allocated. */
octax_status octax_info(octax_env *e, uint64_t out4[4]);

void octax_destroy(octax_env *e);
const char *octax_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* OCTAX_H */
