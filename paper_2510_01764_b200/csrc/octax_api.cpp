// octax_api.cpp -- host side of the C ABI declared in include/octax.h.
//
// Validation of the ROM and game spec (P:140 ROM at 0x200, <= 3584 bytes;
// P:146-158 spec fields), compilation of the score / termination expressions
// to postfix bytecode for the device evaluator, device allocation
// of the structure-of-arrays VM state, and stream-ordered launches.  No torch
// types; plain pointers only.  Independent of oracle/ (own parser, own font).
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/octax.h"
#include "octax_dev.cuh"

namespace octax {
size_t smem_bytes();
cudaError_t launch_step(const StepParams &p, int mode, const int32_t *actions, uint8_t *obs, float *reward,
                        uint8_t *done, uint8_t *term, uint8_t *trunc, cudaStream_t stream);
cudaError_t launch_gen_actions(uint64_t n, uint64_t env_offset, uint64_t aseed, uint64_t t, uint32_t n_actions,
                               int32_t *out, cudaStream_t stream);
cudaError_t launch_expand_obs(uint64_t n, const uint8_t *packed, uint8_t *dense, cudaStream_t stream,
                              const uint8_t *row_mask = nullptr);
cudaError_t launch_get_states(const StepParams &p, const uint64_t *ids, uint64_t count, uint8_t *out,
                              cudaStream_t stream);
cudaError_t launch_state_digests(const StepParams &p, uint64_t first, uint64_t count, uint8_t *canon,
                                 uint64_t *out, cudaStream_t stream);
cudaError_t launch_set_state(const StepParams &p, uint64_t env, const uint8_t *canon, cudaStream_t stream);
}  // namespace octax

using namespace octax;

static thread_local std::string g_last_error;

static octax_status set_err(octax_status s, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return s;
}

static octax_status cuda_err(cudaError_t e, const char *what) {
  return set_err(e == cudaErrorMemoryAllocation ? OCTAX_E_OOM : OCTAX_E_CUDA, "%s: %s", what,
                 cudaGetErrorString(e));
}

#define CU(call, what)                                  \
  do {                                                  \
    cudaError_t _e = (call);                            \
    if (_e != cudaSuccess) return cuda_err(_e, what);   \
  } while (0)

extern "C" const char *octax_last_error(void) { return g_last_error.c_str(); }

// ------------------------------------------------------------------ expression compiler
// Tokenise, then precedence-climb directly to postfix bytecode.  Grammar: C
// operator precedence over u32: || && | ^ & (== !=) (< <= > >=)
// (<< >>) (+ -) (* / // %) unary(- ! ~) primary.  Primaries: decimal / 0x
// literals, V0..V15, VA..VF, V[n], I, DT, ST, mem[e] / memory[e], (e).
namespace {

enum TokKind { T_NUM, T_REG, T_I, T_DT, T_ST, T_MEM, T_OP, T_LP, T_RP, T_LB, T_RB, T_END };

struct Tok {
  TokKind k;
  uint32_t v;
  std::string op;
  size_t at;
};

struct Compiler {
  std::vector<Tok> toks;
  size_t i = 0;
  std::vector<ExprInsn> out;
  int depth = 0, max_depth = 0;
  bool bad = false;
  size_t bad_at = 0;
  std::string msg;

  void fail(size_t at, const std::string &m) {
    if (!bad) { bad = true; bad_at = at; msg = m; }
  }

  static bool ident(char c) { return isalnum((unsigned char)c) || c == '_'; }

  void lex(const char *s) {
    size_t n = strlen(s), p = 0;
    while (p < n && !bad) {
      char c = s[p];
      if (isspace((unsigned char)c)) { ++p; continue; }
      size_t at = p;
      if (isdigit((unsigned char)c)) {
        size_t q = p;
        unsigned long long v = 0;
        bool hex = c == '0' && (s[p + 1] == 'x' || s[p + 1] == 'X');
        if (hex) {
          q = p + 2;
          size_t st = q;
          while (isxdigit((unsigned char)s[q])) {
            v = v * 16 + (isdigit((unsigned char)s[q]) ? s[q] - '0' : (tolower(s[q]) - 'a' + 10));
            if (v > 0xFFFFFFFFull) { fail(at, "literal out of range"); return; }
            ++q;
          }
          if (q == st) { fail(at, "bad hex literal"); return; }
        } else {
          while (isdigit((unsigned char)s[q])) {
            v = v * 10 + (s[q] - '0');
            if (v > 0xFFFFFFFFull) { fail(at, "literal out of range"); return; }
            ++q;
          }
        }
        if (ident(s[q])) { fail(at, "bad literal"); return; }
        toks.push_back({T_NUM, (uint32_t)v, "", at});
        p = q;
        continue;
      }
      if (isalpha((unsigned char)c) || c == '_') {
        size_t q = p;
        while (ident(s[q])) ++q;
        std::string w(s + p, q - p);
        for (auto &ch : w) ch = (char)tolower(ch);
        if (w == "v" && s[q] == '[') {
          size_t r = q + 1;
          while (isspace((unsigned char)s[r])) ++r;
          unsigned long long v = 0;
          size_t st = r;
          bool hex = s[r] == '0' && (s[r + 1] == 'x' || s[r + 1] == 'X');
          if (hex) { r += 2; st = r; while (isxdigit((unsigned char)s[r])) { v = v * 16 + (isdigit((unsigned char)s[r]) ? s[r] - '0' : tolower(s[r]) - 'a' + 10); ++r; if (v > 15) break; } }
          else { while (isdigit((unsigned char)s[r])) { v = v * 10 + (s[r] - '0'); ++r; if (v > 15) break; } }
          if (r == st || v > 15) { fail(at, "bad register index"); return; }
          while (isspace((unsigned char)s[r])) ++r;
          if (s[r] != ']') { fail(r, "expected ']'"); return; }
          toks.push_back({T_REG, (uint32_t)v, "", at});
          p = r + 1;
          continue;
        }
        if (w.size() >= 2 && w[0] == 'v') {
          std::string rest = w.substr(1);
          bool dec = rest.find_first_not_of("0123456789") == std::string::npos;
          if (dec && rest.size() <= 2 && atoi(rest.c_str()) <= 15) {
            toks.push_back({T_REG, (uint32_t)atoi(rest.c_str()), "", at});
            p = q;
            continue;
          }
          if (rest.size() == 1 && rest[0] >= 'a' && rest[0] <= 'f') {
            toks.push_back({T_REG, (uint32_t)(rest[0] - 'a' + 10), "", at});
            p = q;
            continue;
          }
          fail(at, "bad register name");
          return;
        }
        if (w == "i") toks.push_back({T_I, 0, "", at});
        else if (w == "dt") toks.push_back({T_DT, 0, "", at});
        else if (w == "st") toks.push_back({T_ST, 0, "", at});
        else if (w == "mem" || w == "memory") toks.push_back({T_MEM, 0, "", at});
        else { fail(at, "unknown identifier"); return; }
        p = q;
        continue;
      }
      static const char *ops[] = {"||", "&&", "==", "!=", "<=", ">=", "<<", ">>", "//", "|", "^", "&",
                                  "<",  ">",  "+",  "-",  "*",  "/",  "%",  "!",  "~"};
      bool matched = false;
      for (const char *o : ops) {
        size_t L = strlen(o);
        if (strncmp(s + p, o, L) == 0) {
          toks.push_back({T_OP, 0, o, at});
          p += L;
          matched = true;
          break;
        }
      }
      if (matched) continue;
      if (c == '(') { toks.push_back({T_LP, 0, "", at}); ++p; continue; }
      if (c == ')') { toks.push_back({T_RP, 0, "", at}); ++p; continue; }
      if (c == '[') { toks.push_back({T_LB, 0, "", at}); ++p; continue; }
      if (c == ']') { toks.push_back({T_RB, 0, "", at}); ++p; continue; }
      fail(at, "unexpected character");
      return;
    }
    toks.push_back({T_END, 0, "", n});
  }

  void emit(uint8_t op, uint8_t arg = 0, uint32_t imm = 0) {
    out.push_back({op, arg, 0, imm});
    if (op <= X_ST) { ++depth; if (depth > max_depth) max_depth = depth; }
    else if (op >= X_MUL) --depth;
  }

  static int prec(const std::string &o) {
    if (o == "||") return 1;
    if (o == "&&") return 2;
    if (o == "|") return 3;
    if (o == "^") return 4;
    if (o == "&") return 5;
    if (o == "==" || o == "!=") return 6;
    if (o == "<" || o == "<=" || o == ">" || o == ">=") return 7;
    if (o == "<<" || o == ">>") return 8;
    if (o == "+" || o == "-") return 9;
    if (o == "*" || o == "/" || o == "//" || o == "%") return 10;
    return 0;
  }

  static uint8_t binop(const std::string &o) {
    if (o == "||") return X_LOR;
    if (o == "&&") return X_LAND;
    if (o == "|") return X_OR;
    if (o == "^") return X_XOR;
    if (o == "&") return X_AND;
    if (o == "==") return X_EQ;
    if (o == "!=") return X_NE;
    if (o == "<") return X_LT;
    if (o == "<=") return X_LE;
    if (o == ">") return X_GT;
    if (o == ">=") return X_GE;
    if (o == "<<") return X_SHL;
    if (o == ">>") return X_SHR;
    if (o == "+") return X_ADD;
    if (o == "-") return X_SUB;
    if (o == "*") return X_MUL;
    if (o == "%") return X_MOD;
    return X_DIV;  // "/" and "//"
  }

  void unary() {
    if (bad) return;
    const Tok &t = toks[i];
    if (t.k == T_OP && (t.op == "-" || t.op == "!" || t.op == "~")) {
      ++i;
      unary();
      emit(t.op == "-" ? X_NEG : t.op == "!" ? X_NOT : X_BNOT);
      return;
    }
    switch (t.k) {
      case T_NUM: ++i; emit(X_CONST, 0, t.v); return;
      case T_REG: ++i; emit(X_V, (uint8_t)t.v); return;
      case T_I: ++i; emit(X_I); return;
      case T_DT: ++i; emit(X_DT); return;
      case T_ST: ++i; emit(X_ST); return;
      case T_MEM:
        ++i;
        if (toks[i].k != T_LB) { fail(toks[i].at, "expected '['"); return; }
        ++i;
        binary(1);
        if (bad) return;
        if (toks[i].k != T_RB) { fail(toks[i].at, "expected ']'"); return; }
        ++i;
        emit(X_MEM);
        return;
      case T_LP:
        ++i;
        binary(1);
        if (bad) return;
        if (toks[i].k != T_RP) { fail(toks[i].at, "expected ')'"); return; }
        ++i;
        return;
      default:
        fail(t.at, t.k == T_END ? "unexpected end of expression" : "unexpected token");
    }
  }

  void binary(int min_prec) {
    unary();
    while (!bad) {
      const Tok &t = toks[i];
      if (t.k != T_OP) return;
      int pr = prec(t.op);
      if (pr == 0 || pr < min_prec) return;
      ++i;
      binary(pr + 1);  // left associative
      if (bad) return;
      emit(binop(t.op));
    }
  }
};

octax_status compile_expr(const char *src, const char *what, Program &prog) {
  if (!src) return set_err(OCTAX_E_SPEC, "%s is NULL", what);
  Compiler c;
  c.lex(src);
  if (!c.bad) {
    c.binary(1);
    if (!c.bad && c.toks[c.i].k != T_END) c.fail(c.toks[c.i].at, "unexpected trailing input");
  }
  if (c.bad) return set_err(OCTAX_E_EXPR, "%s: %s at byte %zu", what, c.msg.c_str(), c.bad_at);
  // peephole: "V[n] c /" and "V[n] c %" become one push of V[n] / c (% c) by multiply-shift;
  // the byte V[n] < 256 makes q = (V * (2^16 / c + 1)) >> 16 exact for every c <= 255 (error
  // < V / 2^16 < 1 / c); c > 255 gives q = 0; c = 0 keeps x / 0 = x % 0 = 0 (A28)
  {
    std::vector<ExprInsn> o;
    for (size_t k = 0; k < c.out.size(); ++k) {
      if (k + 2 < c.out.size() && c.out[k].op == X_V && c.out[k + 1].op == X_CONST &&
          (c.out[k + 2].op == X_DIV || c.out[k + 2].op == X_MOD)) {
        const uint32_t d = c.out[k + 1].imm;
        ExprInsn f{};
        if (d == 0) {
          f.op = X_CONST;
        } else {
          f.op = c.out[k + 2].op == X_DIV ? X_VDIV : X_VMOD;
          f.arg = c.out[k].arg;
          f.pad = (uint16_t)(d > 255u ? 256u : d);  // only used when d <= 255 (q = 0 above)
          f.imm = d > 255u ? 0u : 65536u / d + 1u;
        }
        o.push_back(f);
        k += 2;
        continue;
      }
      o.push_back(c.out[k]);
    }
    c.out.swap(o);
  }
  if (c.out.size() > (size_t)kMaxOps)
    return set_err(OCTAX_E_EXPR, "%s: expression longer than %u ops", what, (unsigned)kMaxOps);
  if (c.max_depth > kMaxDepth)
    return set_err(OCTAX_E_EXPR, "%s: expression deeper than %u", what, (unsigned)kMaxDepth);
  memset(&prog, 0, sizeof prog);
  for (size_t k = 0; k < c.out.size(); ++k) prog.ops[k] = c.out[k];
  prog.len = (uint32_t)c.out.size();
  prog.depth = (uint32_t)c.max_depth;
  const ExprInsn *o = prog.ops;
  if (prog.len == 1 && o[0].op == X_CONST) {
    prog.kind = 1; prog.ka = o[0].imm;                      // "0"
  } else if (prog.len == 1 && o[0].op == X_V) {
    prog.kind = 2; prog.ka = o[0].arg;                      // "V5"
  } else if (prog.len == 3 && o[0].op == X_V && o[1].op == X_CONST && (o[2].op == X_EQ || o[2].op == X_NE)) {
    prog.kind = o[2].op == X_EQ ? 3u : 4u;                  // "V14 == 0", "V3 != 1"
    prog.ka = o[0].arg; prog.kb = o[1].imm;
  }
  return OCTAX_OK;
}

// Decode table for the kernel core (see octax_dev.cuh).  Built from the ISA
// definition (S:158 opcode list; readings A14/A20) with the quirk bits
// folded in.
void build_desc_table(uint32_t quirks, uint32_t out[kDescEntries]) {
  for (uint32_t k = 0; k < kDescEntries; ++k) out[k] = 0;
  for (uint32_t hi = 0; hi < 14; ++hi)
    for (uint32_t n = 0; n < 16; ++n) {
      uint32_t d = 0;
      switch (hi) {
        case 0x0: d = D_OK; break;  // 00E0 / 00EE / 0NNN decided from the full word
        case 0x1: d = D_OK | D_PCJ; break;
        case 0x2: d = D_OK | D_PCJ | D_CALL; break;
        case 0x3: d = D_OK | D_SKIP; break;
        case 0x4: d = D_OK | D_SKIP | D_SINV; break;
        case 0x5: d = n == 0 ? (D_OK | D_SKIP | D_BVY) : 0u; break;
        case 0x6: d = D_OK | D_WVX; break;
        case 0x7: d = D_OK | D_WVX | D_VSADD; break;
        case 0x8:
          if (n <= 7 || n == 0xE) {
            d = D_OK | D_WVX | D_VSALU;
            if (n >= 4 || ((quirks & OCTAX_Q_VF_RESET) && n >= 1)) d |= D_WVF;
          }
          break;
        case 0x9: d = n == 0 ? (D_OK | D_SKIP | D_SINV | D_BVY) : 0u; break;
        case 0xA: d = D_OK | D_INNN; break;
        case 0xB: d = D_OK | D_BJMP; break;
        case 0xC: d = D_OK | D_RND; break;
        case 0xD: d = D_OK | D_DRAW; break;
      }
      out[(hi << 4) | n] = d;
    }
  struct { uint32_t op; uint32_t d; } ef[] = {
      {0xE09E, D_SKIP | D_SKEY}, {0xE0A1, D_SKIP | D_SKEY | D_SINV}, {0xF007, D_WVX | D_VSDT}, {0xF00A, D_WAIT},
      {0xF015, D_DTW},     {0xF018, D_STW},      {0xF01E, D_IADD},         {0xF029, D_IFONT},
      {0xF033, D_MEM},     {0xF055, D_MEM},      {0xF065, D_MEM}};
  for (auto &e : ef) out[desc_index(e.op)] = D_OK | D_YCHK | e.d | (((e.op >> 4) & 15u) << 28);
}

// Canonical CHIP-8 font, 16 glyphs x 5 rows, stored at 0x050 (A23).
const uint8_t kFont[80] = {
    0xF0, 0x90, 0x90, 0x90, 0xF0, 0x20, 0x60, 0x20, 0x20, 0x70, 0xF0, 0x10, 0xF0, 0x80, 0xF0, 0xF0,
    0x10, 0xF0, 0x10, 0xF0, 0x90, 0x90, 0xF0, 0x10, 0x10, 0xF0, 0x80, 0xF0, 0x10, 0xF0, 0xF0, 0x80,
    0xF0, 0x90, 0xF0, 0xF0, 0x10, 0x20, 0x40, 0x40, 0xF0, 0x90, 0xF0, 0x90, 0xF0, 0xF0, 0x90, 0xF0,
    0x10, 0xF0, 0xF0, 0x90, 0xF0, 0x90, 0x90, 0xE0, 0x90, 0xE0, 0x90, 0xE0, 0xF0, 0x80, 0x80, 0x80,
    0xF0, 0xE0, 0x90, 0x90, 0x90, 0xE0, 0xF0, 0x80, 0xF0, 0x80, 0xF0, 0xF0, 0x80, 0xF0, 0x80, 0x80};

}  // namespace

// ------------------------------------------------------------------ handle
struct octax_env {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint64_t n = 0, env_offset = 0, total = 0;
  StepParams p{};
  uint32_t obs_format = 0, obs_bytes = 1024;
  void *block = nullptr;          // one allocation holding all per-env state
  size_t block_bytes = 0;
  uint8_t *packed_scratch = nullptr;  // packed obs staging for the bool format
  uint8_t *final_scratch = nullptr;   // packed final-obs staging for the bool format (lazy)
  uint8_t *roll_scratch = nullptr;    // packed [T][n] obs staging of bool-format rollouts (lazy)
  uint64_t roll_scratch_bytes = 0;
  // host-step staging (lazy)
  int32_t *d_actions = nullptr;
  uint8_t *d_obs = nullptr;
  float *d_reward = nullptr;
  uint8_t *d_flags = nullptr;  // done | term | trunc, 3*n
  uint8_t *d_frame = nullptr;  // [n][256] newest display (octax_step_host_frame)
  cudaStream_t copy_stream = nullptr;           // host steps: device -> host copies of finished chunks
  cudaEvent_t chunk_done[kMaxHostChunks] = {};  // one per chunk launch
  // get/set state staging (lazy)
  uint64_t *d_ids = nullptr;
  uint8_t *d_canon = nullptr;
  uint64_t canon_cap = 0;
};

static void free_env(octax_env *e) {
  if (!e) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(e->device);
  cudaFree(e->block);
  cudaFree(e->packed_scratch);
  cudaFree(e->final_scratch);
  cudaFree(e->roll_scratch);
  cudaFree(e->d_actions);
  cudaFree(e->d_obs);
  cudaFree(e->d_reward);
  cudaFree(e->d_flags);
  cudaFree(e->d_frame);
  if (e->copy_stream) {
    cudaStreamDestroy(e->copy_stream);
    for (auto ev : e->chunk_done)
      if (ev) cudaEventDestroy(ev);
  }
  cudaFree(e->d_ids);
  cudaFree(e->d_canon);
  cudaSetDevice(prev);
  delete e;
}

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int d) { cudaGetDevice(&prev); if (prev != d) cudaSetDevice(d); }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

extern "C" octax_status octax_create(const uint8_t *rom, size_t rom_len, const octax_game_spec *spec,
                                     uint64_t n_envs, uint64_t seed, const octax_device_opts *opts,
                                     octax_env **out) {
  if (!out) return set_err(OCTAX_E_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (!spec) return set_err(OCTAX_E_INVALID_ARG, "spec is NULL");
  if (!rom || rom_len == 0) return set_err(OCTAX_E_ROM_EMPTY, "ROM is empty");
  if (rom_len > 4096 - 0x200) return set_err(OCTAX_E_ROM_TOO_LARGE, "ROM of %zu bytes > 3584", rom_len);
  if (spec->abi_version != OCTAX_ABI_VERSION) return set_err(OCTAX_E_SPEC, "abi_version must be 1");
  if (n_envs == 0) return set_err(OCTAX_E_INVALID_ARG, "n_envs must be > 0");
  if (n_envs > (1ull << 31)) return set_err(OCTAX_E_INVALID_ARG, "n_envs too large");
  if (spec->frame_skip == 0) return set_err(OCTAX_E_SPEC, "frame_skip must be > 0");
  if (spec->instructions_per_frame == 0) return set_err(OCTAX_E_SPEC, "instructions_per_frame must be > 0");
  if (spec->n_action_keys < 1 || spec->n_action_keys > 16 || !spec->action_keys)
    return set_err(OCTAX_E_SPEC, "n_action_keys must be in 1..16");
  uint32_t seen = 0;
  for (uint32_t k = 0; k < spec->n_action_keys; ++k) {
    if (spec->action_keys[k] > 15) return set_err(OCTAX_E_SPEC, "action key %u > 15", spec->action_keys[k]);
    if (seen & (1u << spec->action_keys[k])) return set_err(OCTAX_E_SPEC, "duplicate action key %u", spec->action_keys[k]);
    seen |= 1u << spec->action_keys[k];
  }
  if (spec->n_startup > kMaxStartup) return set_err(OCTAX_E_SPEC, "more than %u startup segments", kMaxStartup);
  if (spec->n_startup && !spec->startup) return set_err(OCTAX_E_SPEC, "startup is NULL");
  if (spec->quirks & ~31u) return set_err(OCTAX_E_SPEC, "unknown quirk bits");
  if (spec->obs_format & ~(uint32_t)(1 | OCTAX_OBS_STACK_FRAMES)) return set_err(OCTAX_E_SPEC, "unknown obs_format");

  octax_env *e = new octax_env();
  StepParams &p = e->p;
  octax_status st = compile_expr(spec->score_expr, "score_expr", p.score);
  if (st == OCTAX_OK) st = compile_expr(spec->terminated_expr, "terminated_expr", p.term);
  if (st != OCTAX_OK) { delete e; return st; }

  e->device = opts ? opts->device : 0;
  e->stream = opts ? (cudaStream_t)opts->cuda_stream : nullptr;
  e->n = n_envs;
  e->env_offset = opts ? opts->env_offset : 0;
  e->total = (opts && opts->total_envs) ? opts->total_envs : n_envs;
  e->obs_format = spec->obs_format & 1u;  // layout; the stacking flag goes to the kernel
  e->obs_bytes = e->obs_format == OCTAX_OBS_PACKED ? 1024 : 8192;

  p.n = n_envs;
  p.env_offset = e->env_offset;
  p.frame_skip = spec->frame_skip;
  p.ipf = spec->instructions_per_frame;
  p.max_steps = spec->max_episode_steps;
  p.quirks = spec->quirks;
  p.obs_format = spec->obs_format & 1u;
  p.stack_frames = (spec->obs_format & OCTAX_OBS_STACK_FRAMES) ? 1u : 0u;
  p.n_actions = spec->n_action_keys + 1;
  p.keymask[0] = 0;
  for (uint32_t k = 0; k < spec->n_action_keys; ++k) p.keymask[k + 1] = (uint16_t)(1u << spec->action_keys[k]);
  p.n_startup = spec->n_startup;
  for (uint32_t k = 0; k < spec->n_startup; ++k) {
    p.startup_keys[k] = spec->startup[k].keymask;
    p.startup_frames[k] = spec->startup[k].frames;
  }

  DeviceGuard g(e->device);
  // one allocation: image | stats | regs | ctrl | book | stack | dirty | ring | ram
  const uint64_t n = n_envs;
  size_t off = 0;
  auto carve = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~size_t(255); return o; };
  size_t o_img = carve(kStageBytes), o_dec = carve(8 * kDecEntries), o_words = carve(2 * kWordEntries), o_stats = carve(64), o_regs = carve(16 * n), o_ctrl = carve(16 * n),
         o_book = carve(16 * n), o_stack = carve(32 * n), o_dirty = carve(8 * n),
         o_ring = carve(1024 * ((n + kBlock - 1) / kBlock * kBlock)),
         o_ram = carve(4096 * n);
  // deferred-reset list (only for specs with startup segments)
  const size_t o_rcnt = spec->n_startup ? carve(4) : 0, o_rids = spec->n_startup ? carve(4 * n) : 0;
  e->block_bytes = off;
  cudaError_t ce = cudaMalloc(&e->block, off);
  if (ce != cudaSuccess) { free_env(e); return cuda_err(ce, "cudaMalloc(state)"); }
  uint8_t *base = (uint8_t *)e->block;
  p.s.image = base + o_img;
  p.s.dec = (const uint2 *)(base + o_dec);
  p.s.words = (const uint16_t *)(base + o_words);
  p.s.stats = (unsigned long long *)(base + o_stats);
  p.s.regs = (uint4 *)(base + o_regs);
  p.s.ctrl = (uint4 *)(base + o_ctrl);
  p.s.book = (uint4 *)(base + o_book);
  p.s.stack = (uint4 *)(base + o_stack);
  p.s.dirty = (uint64_t *)(base + o_dirty);
  p.s.ring = (uint64_t *)(base + o_ring);
  p.s.ring_stride = (n + kBlock - 1) / kBlock * kBlock * 32;
  p.s.ram = base + o_ram;
  p.reset_count = spec->n_startup ? (uint32_t *)(base + o_rcnt) : nullptr;
  p.reset_ids = spec->n_startup ? (uint32_t *)(base + o_rids) : nullptr;
  // state is fully written by the reset kernel; zero the small fields anyway
  ce = cudaMemsetAsync(base, 0, o_ring, e->stream);
  if (ce != cudaSuccess) { free_env(e); return cuda_err(ce, "cudaMemset"); }
  uint8_t image[kStageBytes];
  memset(image, 0, sizeof image);
  memcpy(image + 0x50, kFont, sizeof kFont);
  memcpy(image + 0x200, rom, rom_len);
  const uint32_t *dtab = reinterpret_cast<const uint32_t *>(image + kImageBytes);
  build_desc_table(spec->quirks, const_cast<uint32_t *>(dtab));
  std::vector<uint2> dec(kDecEntries);
  for (uint32_t pc = 0; pc < kDecEntries; ++pc) {
    if (pc <= 0xFFEu) {
      make_entry(((uint32_t)image[pc] << 8) | image[pc + 1], dtab, spec->quirks, dec[pc].x, dec[pc].y);
    } else {
      dec[pc] = make_uint2(E_BAD, 1u << 18);  // fetch past 0xFFE halts (A17); SP delta 0
    }
  }
  ce = cudaMemcpyAsync(base + o_img, image, kStageBytes, cudaMemcpyHostToDevice, e->stream);
  if (ce == cudaSuccess)
    ce = cudaMemcpyAsync(base + o_dec, dec.data(), 8 * kDecEntries, cudaMemcpyHostToDevice, e->stream);
  // one entry per 16-bit PC (stored PCs are 16-bit), so the warp kernel's fetch needs no clamp;
  // every PC past 0xFFE holds 0x5001, an invalid word: the kernel halts (A17)
  std::vector<uint16_t> words(kWordEntries, 0x5001);
  for (uint32_t pc = 0; pc < kImageBytes - 1; ++pc) words[pc] = (uint16_t)((image[pc] << 8) | image[pc + 1]);
  if (ce == cudaSuccess)
    ce = cudaMemcpyAsync(base + o_words, words.data(), 2 * kWordEntries, cudaMemcpyHostToDevice, e->stream);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(e->stream);
  if (ce != cudaSuccess) { free_env(e); return cuda_err(ce, "upload image"); }
  if (e->obs_format != OCTAX_OBS_PACKED) {
    ce = cudaMalloc(&e->packed_scratch, 1024 * n);
    if (ce != cudaSuccess) { free_env(e); return cuda_err(ce, "cudaMalloc(obs scratch)"); }
  }
  octax_set_kernel(e, OCTAX_KERNEL_AUTO);
  st = octax_reset(e, seed, nullptr);
  if (st != OCTAX_OK) { free_env(e); return st; }
  *out = e;
  return OCTAX_OK;
}

extern "C" octax_status octax_reset(octax_env *e, uint64_t seed, void *obs_out) {
  if (!e) return set_err(OCTAX_E_INVALID_ARG, "env is NULL");
  DeviceGuard g(e->device);
  e->p.seed = seed;
  e->p.head = 0;
  CU(cudaMemsetAsync(e->p.s.stats, 0, 32, e->stream), "reset stats");
  uint8_t *packed = (uint8_t *)obs_out;
  if (obs_out && e->obs_format != OCTAX_OBS_PACKED) packed = e->packed_scratch;
  CU(launch_step(e->p, MODE_RESET, nullptr, packed, nullptr, nullptr, nullptr, nullptr, e->stream), "reset kernel");
  if (obs_out && e->obs_format != OCTAX_OBS_PACKED)
    CU(launch_expand_obs(e->n, packed, (uint8_t *)obs_out, e->stream), "expand obs");
  return OCTAX_OK;
}

extern "C" octax_status octax_step_ex(octax_env *e, const int32_t *actions, void *obs_out, float *reward_out,
                                      uint8_t *done_out, uint8_t *terminated_out, uint8_t *truncated_out,
                                      const octax_step_extras *extras) {
  if (!e || !actions || !obs_out || !reward_out || !done_out)
    return set_err(OCTAX_E_INVALID_ARG, "NULL argument to octax_step");
  DeviceGuard g(e->device);
  uint8_t *packed = e->obs_format == OCTAX_OBS_PACKED ? (uint8_t *)obs_out : e->packed_scratch;
  StepParams p = e->p;
  p.final_obs = nullptr;
  p.frame_out = nullptr;
  p.ep_ret_out = nullptr;
  p.ep_len_out = nullptr;
  if (extras) {
    p.frame_out = (uint8_t *)extras->frame_out;
    p.ep_ret_out = extras->episode_return_out;
    p.ep_len_out = extras->episode_length_out;
    if (extras->final_obs_out) {
      if (e->obs_format == OCTAX_OBS_PACKED) {
        p.final_obs = (uint8_t *)extras->final_obs_out;
      } else {
        if (!e->final_scratch) CU(cudaMalloc(&e->final_scratch, 1024 * e->n), "cudaMalloc(final obs scratch)");
        p.final_obs = e->final_scratch;
      }
    }
  }
  CU(launch_step(p, MODE_STEP, actions, packed, reward_out, done_out, terminated_out, truncated_out, e->stream),
     "step kernel");
  if (e->obs_format != OCTAX_OBS_PACKED) {
    CU(launch_expand_obs(e->n, packed, (uint8_t *)obs_out, e->stream), "expand obs");
    if (p.final_obs)
      CU(launch_expand_obs(e->n, p.final_obs, (uint8_t *)extras->final_obs_out, e->stream, done_out), "expand final obs");
  }
  e->p.head = (e->p.head + 1) & 3u;
  return OCTAX_OK;
}

// Host-buffer step, pipelined: the envs are stepped in `chunks` launches of consecutive CTA blocks
// on the handle's stream, and each chunk's results go device -> host on a second stream as soon
// as its launch is done, so the PCIe copy of chunk c overlaps the kernel of chunk c+1 (the copy,
// not the kernel, bounds a host step: ~1 GB of obs vs a 0.5 ms kernel at 1M envs).  frame: copy
// the newest display ([n][256], extras.frame_out) instead of the 4-plane obs.
static octax_status host_step(octax_env *e, bool frame, const int32_t *actions_host, void *out_host,
                              float *reward_host, uint8_t *done_host, uint8_t *terminated_host,
                              uint8_t *truncated_host) {
  DeviceGuard g(e->device);
  const uint64_t n = e->n;
  if (!e->d_actions) {
    CU(cudaMalloc(&e->d_actions, 4 * n), "cudaMalloc");
    CU(cudaMalloc(&e->d_obs, (size_t)e->obs_bytes * n), "cudaMalloc");
    CU(cudaMalloc(&e->d_reward, 4 * n), "cudaMalloc");
    CU(cudaMalloc(&e->d_flags, 3 * n), "cudaMalloc");
  }
  if (frame && !e->d_frame) CU(cudaMalloc(&e->d_frame, 256 * n), "cudaMalloc(frame)");
  if (!e->copy_stream) {
    CU(cudaStreamCreateWithFlags(&e->copy_stream, cudaStreamNonBlocking), "copy stream");
    for (auto &ev : e->chunk_done) CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
  }
  CU(cudaMemcpyAsync(e->d_actions, actions_host, 4 * n, cudaMemcpyHostToDevice, e->stream), "H2D actions");
  const uint32_t nblocks = (uint32_t)((n + kBlock - 1) / kBlock);
  // chunks: a launch per >= one wave of CTAs (148 SMs x 5), at most kMaxHostChunks: the first
  // chunk's kernel is the only compute not hidden behind a copy (A/B at 1M envs: 1 chunk 1.73e8,
  // 2 chunks 1.93e8, 5 chunks 2.02e8 env steps/s through octax_step_host_frame)
  uint32_t chunks = nblocks / 740u;
  chunks = chunks < 1u ? 1u : (chunks > kMaxHostChunks ? kMaxHostChunks : chunks);
  uint8_t *packed = e->obs_format == OCTAX_OBS_PACKED ? e->d_obs : e->packed_scratch;
  const size_t ob = e->obs_bytes;
  for (uint32_t c = 0; c < chunks; ++c) {
    const uint32_t b0 = (uint32_t)((uint64_t)nblocks * c / chunks), b1 = (uint32_t)((uint64_t)nblocks * (c + 1) / chunks);
    const uint64_t e0 = (uint64_t)b0 * kBlock, e1 = (uint64_t)b1 * kBlock < n ? (uint64_t)b1 * kBlock : n;
    StepParams p = e->p;
    p.final_obs = nullptr;
    p.frame_out = frame ? e->d_frame : nullptr;
    p.ep_ret_out = nullptr;
    p.ep_len_out = nullptr;
    p.block_base = b0;
    p.block_count = b1 - b0;
    CU(launch_step(p, MODE_STEP, e->d_actions, packed, e->d_reward, e->d_flags, e->d_flags + n, e->d_flags + 2 * n,
                   e->stream), "step kernel");
    if (e->obs_format != OCTAX_OBS_PACKED && !frame)
      CU(launch_expand_obs(e1 - e0, packed + e0 * 1024, e->d_obs + e0 * ob, e->stream), "expand obs");
    CU(cudaEventRecord(e->chunk_done[c], e->stream), "event record");
    CU(cudaStreamWaitEvent(e->copy_stream, e->chunk_done[c], 0), "stream wait");
    const uint64_t m = e1 - e0;
    if (frame)
      CU(cudaMemcpyAsync((uint8_t *)out_host + e0 * 256, e->d_frame + e0 * 256, 256 * m, cudaMemcpyDeviceToHost,
                         e->copy_stream), "D2H frame");
    else
      CU(cudaMemcpyAsync((uint8_t *)out_host + e0 * ob, e->d_obs + e0 * ob, ob * m, cudaMemcpyDeviceToHost,
                         e->copy_stream), "D2H obs");
  }
  // the small per-env outputs (5 B/env) once, after the last chunk: per-copy overhead, not bytes,
  // is their cost
  CU(cudaMemcpyAsync(reward_host, e->d_reward, 4 * n, cudaMemcpyDeviceToHost, e->copy_stream), "D2H reward");
  CU(cudaMemcpyAsync(done_host, e->d_flags, n, cudaMemcpyDeviceToHost, e->copy_stream), "D2H done");
  if (terminated_host)
    CU(cudaMemcpyAsync(terminated_host, e->d_flags + n, n, cudaMemcpyDeviceToHost, e->copy_stream), "D2H term");
  if (truncated_host)
    CU(cudaMemcpyAsync(truncated_host, e->d_flags + 2 * n, n, cudaMemcpyDeviceToHost, e->copy_stream), "D2H trunc");
  e->p.head = (e->p.head + 1) & 3u;
  CU(cudaStreamSynchronize(e->copy_stream), "sync");
  CU(cudaStreamSynchronize(e->stream), "sync");
  return OCTAX_OK;
}

extern "C" octax_status octax_step(octax_env *e, const int32_t *actions, void *obs_out, float *reward_out,
                                   uint8_t *done_out, uint8_t *terminated_out, uint8_t *truncated_out) {
  return octax_step_ex(e, actions, obs_out, reward_out, done_out, terminated_out, truncated_out, nullptr);
}

extern "C" octax_status octax_step_host(octax_env *e, const int32_t *actions_host, void *obs_host,
                                        float *reward_host, uint8_t *done_host, uint8_t *terminated_host,
                                        uint8_t *truncated_host) {
  if (!e || !actions_host || !obs_host || !reward_host || !done_host)
    return set_err(OCTAX_E_INVALID_ARG, "NULL argument to octax_step_host");
  return host_step(e, false, actions_host, obs_host, reward_host, done_host, terminated_host, truncated_host);
}

extern "C" octax_status octax_step_host_frame(octax_env *e, const int32_t *actions_host, void *frame_host,
                                              float *reward_host, uint8_t *done_host, uint8_t *terminated_host,
                                              uint8_t *truncated_host) {
  if (!e || !actions_host || !frame_host || !reward_host || !done_host)
    return set_err(OCTAX_E_INVALID_ARG, "NULL argument to octax_step_host_frame");
  return host_step(e, true, actions_host, frame_host, reward_host, done_host, terminated_host, truncated_host);
}

extern "C" octax_status octax_rollout(octax_env *e, uint32_t T, const int32_t *actions, uint64_t aseed, uint64_t t0,
                                      void *obs_out, uint64_t obs_step_stride, float *reward_out, uint8_t *done_out,
                                      uint8_t *terminated_out, uint8_t *truncated_out, uint64_t out_step_stride) {
  if (!e || !reward_out || !done_out)
    return set_err(OCTAX_E_INVALID_ARG, "NULL argument to octax_rollout");
  if (T == 0) return OCTAX_OK;
  if (obs_step_stride % 16 != 0)
    return set_err(OCTAX_E_INVALID_ARG, "octax_rollout: obs_step_stride must be a multiple of 16 bytes");
  if (!obs_out) obs_step_stride = 0;
  if ((obs_step_stride != 0 && obs_step_stride < (uint64_t)e->obs_bytes * e->n) ||
      (out_step_stride != 0 && out_step_stride < e->n))
    return set_err(OCTAX_E_INVALID_ARG, "octax_rollout: a non-zero step stride must cover all n envs");
  DeviceGuard g(e->device);
  StepParams p = e->p;
  p.final_obs = nullptr;
  p.frame_out = nullptr;
  p.ep_ret_out = nullptr;
  p.ep_len_out = nullptr;
  p.reset_ids = nullptr;  // resets run inline inside the rollout kernel
  p.reset_count = nullptr;
  p.T = T;
  p.aseed = aseed;
  p.t0 = t0;
  p.out_stride = out_step_stride;
  uint8_t *packed = (uint8_t *)obs_out;
  uint64_t planes_out = 0;  // bool layout: packed obs planes to expand after the kernel
  if (obs_out && e->obs_format != OCTAX_OBS_PACKED) {
    // the bool [n,4,64,32] layout: the kernel writes packed obs, expand_obs_kernel expands them
    // after it -- every step's (a [T][n] packed staging buffer) or, with stride 0, the last step's
    if (obs_step_stride == 0) {
      packed = e->packed_scratch;
      planes_out = e->n;
    } else {
      if (obs_step_stride != (uint64_t)e->obs_bytes * e->n)
        return set_err(OCTAX_E_INVALID_ARG, "octax_rollout: bool observations need stride 0 or n * 8192 bytes");
      const uint64_t need = (uint64_t)T * e->n * 1024;
      if (need > e->roll_scratch_bytes) {
        cudaFree(e->roll_scratch);
        e->roll_scratch = nullptr;
        e->roll_scratch_bytes = 0;
        CU(cudaMalloc(&e->roll_scratch, need), "cudaMalloc(rollout obs staging)");
        e->roll_scratch_bytes = need;
      }
      packed = e->roll_scratch;
      planes_out = (uint64_t)T * e->n;
      obs_step_stride = 1024 * e->n;
    }
  }
  p.obs_stride = obs_step_stride / 8;
  CU(launch_step(p, MODE_ROLLOUT, actions, packed, reward_out, done_out, terminated_out, truncated_out, e->stream),
     "rollout kernel");
  if (planes_out) CU(launch_expand_obs(planes_out, packed, (uint8_t *)obs_out, e->stream), "expand obs");
  e->p.head = (e->p.head + T) & 3u;
  return OCTAX_OK;
}

extern "C" octax_status octax_gen_actions(octax_env *e, uint64_t aseed, uint64_t t, int32_t *actions_out) {
  if (!e || !actions_out) return set_err(OCTAX_E_INVALID_ARG, "NULL argument");
  DeviceGuard g(e->device);
  CU(launch_gen_actions(e->n, e->env_offset, aseed, t, e->p.n_actions, actions_out, e->stream), "gen actions");
  return OCTAX_OK;
}

extern "C" octax_status octax_stats(octax_env *e, int64_t out4[4]) {
  if (!e || !out4) return set_err(OCTAX_E_INVALID_ARG, "NULL argument");
  DeviceGuard g(e->device);
  unsigned long long h[4];
  CU(cudaMemcpyAsync(h, e->p.s.stats, 32, cudaMemcpyDeviceToHost, e->stream), "D2H stats");
  CU(cudaStreamSynchronize(e->stream), "sync");
  for (int k = 0; k < 4; ++k) out4[k] = (int64_t)h[k];
  if (h[3]) return set_err(OCTAX_E_DEVICE, "out-of-range action seen (treated as no-op)");
  return OCTAX_OK;
}

extern "C" octax_status octax_stats_device(octax_env *e, int64_t *out4_device) {
  if (!e || !out4_device) return set_err(OCTAX_E_INVALID_ARG, "NULL argument");
  DeviceGuard g(e->device);
  CU(cudaMemcpyAsync(out4_device, e->p.s.stats, 32, cudaMemcpyDeviceToDevice, e->stream), "D2D stats");
  return OCTAX_OK;
}

static octax_status ensure_canon(octax_env *e, uint64_t count) {
  if (count <= e->canon_cap) return OCTAX_OK;
  cudaFree(e->d_ids);
  cudaFree(e->d_canon);
  e->d_ids = nullptr;
  e->d_canon = nullptr;
  e->canon_cap = 0;
  CU(cudaMalloc(&e->d_ids, 8 * count), "cudaMalloc");
  CU(cudaMalloc(&e->d_canon, (size_t)OCTAX_CANON_BYTES * count), "cudaMalloc");
  e->canon_cap = count;
  return OCTAX_OK;
}

extern "C" octax_status octax_get_states(octax_env *e, const uint64_t *envs, uint64_t count, uint8_t *canon_out) {
  if (!e || !envs || !canon_out) return set_err(OCTAX_E_INVALID_ARG, "NULL argument");
  if (count == 0) return OCTAX_OK;
  for (uint64_t k = 0; k < count; ++k)
    if (envs[k] >= e->n) return set_err(OCTAX_E_INVALID_ARG, "env index %llu out of range", (unsigned long long)envs[k]);
  DeviceGuard g(e->device);
  octax_status st = ensure_canon(e, count);
  if (st != OCTAX_OK) return st;
  CU(cudaMemcpyAsync(e->d_ids, envs, 8 * count, cudaMemcpyHostToDevice, e->stream), "H2D ids");
  CU(launch_get_states(e->p, e->d_ids, count, e->d_canon, e->stream), "get_states kernel");
  CU(cudaMemcpyAsync(canon_out, e->d_canon, (size_t)OCTAX_CANON_BYTES * count, cudaMemcpyDeviceToHost, e->stream),
     "D2H canon");
  CU(cudaStreamSynchronize(e->stream), "sync");
  return OCTAX_OK;
}

extern "C" octax_status octax_state_digests(octax_env *e, uint64_t first, uint64_t count,
                                            uint64_t *digests_out, uint64_t *sum_out) {
  if (!e || (!digests_out && !sum_out)) return set_err(OCTAX_E_INVALID_ARG, "NULL argument");
  if (first > e->n || count > e->n - first) return set_err(OCTAX_E_INVALID_ARG, "env range out of bounds");
  DeviceGuard g(e->device);
  const uint64_t chunk = count < 65536 ? count : 65536;
  uint64_t sum = 0;
  if (count) {
    octax_status st = ensure_canon(e, chunk);
    if (st != OCTAX_OK) return st;
    std::vector<uint64_t> h(chunk);
    for (uint64_t k = 0; k < count; k += chunk) {
      const uint64_t m = count - k < chunk ? count - k : chunk;
      // d_ids doubles as the digest buffer (8 B per env, chunk entries)
      CU(launch_state_digests(e->p, first + k, m, e->d_canon, e->d_ids, e->stream), "digest kernels");
      CU(cudaMemcpyAsync(h.data(), e->d_ids, 8 * m, cudaMemcpyDeviceToHost, e->stream), "D2H digests");
      CU(cudaStreamSynchronize(e->stream), "sync");
      for (uint64_t q = 0; q < m; ++q) {
        if (digests_out) digests_out[k + q] = h[q];
        sum += h[q];
      }
    }
  }
  if (sum_out) *sum_out = sum;
  return OCTAX_OK;
}

extern "C" octax_status octax_get_state(octax_env *e, uint64_t env, uint8_t *canon_out) {
  return octax_get_states(e, &env, 1, canon_out);
}

extern "C" octax_status octax_set_state(octax_env *e, uint64_t env, const uint8_t *canon_in) {
  if (!e || !canon_in) return set_err(OCTAX_E_INVALID_ARG, "NULL argument");
  if (env >= e->n) return set_err(OCTAX_E_INVALID_ARG, "env index out of range");
  if (canon_in[20] > 16) return set_err(OCTAX_E_INVALID_ARG, "SP > 16");
  DeviceGuard g(e->device);
  octax_status st = ensure_canon(e, 1);
  if (st != OCTAX_OK) return st;
  CU(cudaMemcpyAsync(e->d_canon, canon_in, OCTAX_CANON_BYTES, cudaMemcpyHostToDevice, e->stream), "H2D canon");
  CU(launch_set_state(e->p, env, e->d_canon, e->stream), "set_state kernel");
  CU(cudaStreamSynchronize(e->stream), "sync");
  return OCTAX_OK;
}

static uint64_t warp_auto_max() {
  const char *s = getenv("OCTAX_WARP_AUTO_MAX");
  return s ? strtoull(s, nullptr, 10) : (uint64_t)OCTAX_WARP_AUTO_MAX_ENVS;
}

extern "C" octax_status octax_set_kernel(octax_env *e, int kernel) {
  if (!e) return set_err(OCTAX_E_INVALID_ARG, "NULL handle");
  if (kernel != OCTAX_KERNEL_AUTO && kernel != OCTAX_KERNEL_LANE && kernel != OCTAX_KERNEL_WARP)
    return set_err(OCTAX_E_INVALID_ARG, "kernel must be OCTAX_KERNEL_AUTO, _LANE or _WARP");
  e->p.warp = kernel == OCTAX_KERNEL_WARP || (kernel == OCTAX_KERNEL_AUTO && e->n <= warp_auto_max());
  return OCTAX_OK;
}

extern "C" octax_status octax_get_kernel(octax_env *e, int *kernel_out) {
  if (!e || !kernel_out) return set_err(OCTAX_E_INVALID_ARG, "NULL argument");
  *kernel_out = e->p.warp ? OCTAX_KERNEL_WARP : OCTAX_KERNEL_LANE;
  return OCTAX_OK;
}

extern "C" octax_status octax_info(octax_env *e, uint64_t out4[4]) {
  if (!e || !out4) return set_err(OCTAX_E_INVALID_ARG, "NULL argument");
  out4[0] = e->n;
  out4[1] = e->p.n_actions;
  out4[2] = e->obs_bytes;
  out4[3] = e->block_bytes;
  return OCTAX_OK;
}

extern "C" void octax_destroy(octax_env *e) { free_env(e); }
