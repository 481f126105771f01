/*
 * octax_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU implementation of the batched Octax
 * environment step (arXiv 2510.01764, "Octax: Accelerated CHIP-8 Arcade
 * Environments for RL in JAX").  It exists so that the CUDA path in
 * paper_2510_01764_b200/ can be checked against something independent.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * --impl reference) may load this library.  The product path never does.
 * It shares no code, header, table or constant generator with the CUDA
 * path: the font table, Philox, the expression parser and every opcode
 * handler are written out again here on purpose.
 *
 * Citations: P:n = /root/reference/PAPER.md line n (section named),
 *            S:n = /root/reference/SPEC.md line n (interfaces only),
 *            A<k> = reading k of DESIGN.md "Readings of the paper".
 *
 * Representation (deliberately unlike the GPU path): byte-array RAM of
 * 4096 bytes per env, display as bool[32][64], history as 4 full display
 * copies, expressions as a recursive-descent AST evaluated recursively.
 */
#ifndef OCTAX_ORACLE_H
#define OCTAX_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (same numeric meaning as the product ABI, defined again) */
#define ORACLE_OK 0
#define ORACLE_E_INVALID_ARG (-1)
#define ORACLE_E_ROM_EMPTY (-2)
#define ORACLE_E_ROM_TOO_LARGE (-3)
#define ORACLE_E_SPEC (-4)
#define ORACLE_E_EXPR (-5)
#define ORACLE_E_OOM (-7)
#define ORACLE_E_DEVICE (-8)

/* quirk bits (A14; 0 = the "modern" profile) */
#define ORACLE_Q_SHIFT_VY 1u
#define ORACLE_Q_LOADSTORE_INC_I 2u
#define ORACLE_Q_JUMP_VX 4u
#define ORACLE_Q_WRAP_SPRITES 8u
#define ORACLE_Q_VF_RESET 16u

/* observation formats (A3, A4) */
#define ORACLE_OBS_PACKED 0u      /* u8 [n][4][32][8], MSB = leftmost pixel */
#define ORACLE_OBS_BOOL_XMAJOR 1u /* u8 0/1 [n][4][64][32], paper axis order */
#define ORACLE_OBS_STACK_FRAMES 16u /* flag: stack the last 4 frames of the step */

#define ORACLE_CANON_BYTES 5200u

typedef struct {
  uint16_t keymask;
  uint32_t frames;
} oracle_startup_seg;

typedef struct {
  uint32_t abi_version; /* must be 1 */
  const char *score_expr;
  const char *terminated_expr;
  const uint8_t *action_keys;
  uint32_t n_action_keys;
  const oracle_startup_seg *startup;
  uint32_t n_startup;
  uint32_t frame_skip;
  uint32_t instructions_per_frame;
  uint32_t max_episode_steps;
  uint32_t quirks;
  uint32_t obs_format;
} oracle_game_spec;

typedef struct oracle_env oracle_env;

int octax_oracle_create(const uint8_t *rom, size_t rom_len,
                        const oracle_game_spec *spec, uint64_t n_envs,
                        uint64_t seed, uint64_t env_offset, oracle_env **out);
int octax_oracle_reset(oracle_env *e, uint64_t seed, uint8_t *obs_out);
int octax_oracle_step(oracle_env *e, const int32_t *actions, uint8_t *obs_out,
                      float *reward_out, uint8_t *done_out,
                      uint8_t *terminated_out, uint8_t *truncated_out);
int octax_oracle_step_ex(oracle_env *e, const int32_t *actions, uint8_t *obs_out,
                         float *reward_out, uint8_t *done_out,
                         uint8_t *terminated_out, uint8_t *truncated_out,
                         uint8_t *final_obs_out, int32_t *episode_return_out,
                         uint32_t *episode_length_out);
int octax_oracle_stats(oracle_env *e, int64_t out4[4]);
int octax_oracle_get_state(oracle_env *e, uint64_t env, uint8_t *canon_out);
int octax_oracle_set_state(oracle_env *e, uint64_t env, const uint8_t *canon_in);
void octax_oracle_destroy(oracle_env *e);
const char *octax_oracle_last_error(void);

/* ---- test hooks (machine level, no reward/obs bookkeeping) ---- */
/* Run n single CHIP-8 cycles on env `env` with the key mask `keys` held. */
int octax_oracle_run_cycles(oracle_env *e, uint64_t env, uint32_t n, uint16_t keys);
/* Run n frames (ipf cycles, then the timer tick) with `keys` held. */
int octax_oracle_run_frames(oracle_env *e, uint64_t env, uint32_t n, uint16_t keys);
/* The 60 Hz timer tick of one frame alone, for cycle-level tracing. */
int octax_oracle_tick_timers(oracle_env *e, uint64_t env);
/* Parse + evaluate an expression against a canonical state. */
int octax_oracle_eval_expr(const char *expr, const uint8_t *canon_state,
                           uint32_t *value_out, size_t *err_offset_out);
/* Random123 Philox4x32-10. */
void octax_oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2],
                                uint32_t out[4]);
/* Synthetic benchmark action (SURVEY c.1 "synthetic action"). */
int32_t octax_oracle_synthetic_action(uint64_t aseed, uint64_t t, uint64_t gid,
                                      uint32_t n_actions);
/* Per-env workload trace counters for the last step: opcode class histogram
   (16 classes by op>>12), sprite rows drawn.  out must hold 17 u64. */
int octax_oracle_counters(oracle_env *e, uint64_t env, uint64_t out17[17]);

#ifdef __cplusplus
}
#endif
#endif
