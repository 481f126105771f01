/*
 * octax_oracle.c -- TEST INFRASTRUCTURE ONLY (see octax_oracle.h).
 *
 * Plain single-threaded C11.  Every function follows the normative
 * pseudo-code of SURVEY.md §8(c) c.1, which restates the paper:
 *   machine state ............ P:130, P:140 (§3.1-3.2), P:313-321 (App. A.2)
 *   fetch / decode / execute .. P:142-144 (§3.2), P:325-331 (App. A.3)
 *   DXYN XOR + collision ...... P:144, P:327, P:333 (App. A.3)
 *   timers, frame skip ........ P:146 (§3.2), P:228 (§4.2: 4 frames / step)
 *   score / termination ....... P:152-154 (§3.3), P:1571-1584 (App. D)
 *   obs stacking, actions ..... P:146
 *   startup / auto-reset ...... P:146
 * and the readings A1..A26 listed in DESIGN.md where the paper is silent.
 *
 * Nothing here is blocked, fused, vectorised or reordered: one env at a
 * time, one cycle at a time, one pixel at a time.
 */
#include "octax_oracle.h"

#include <stdbool.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* errors                                                              */
/* ------------------------------------------------------------------ */
static _Thread_local char g_err[512];

static int fail(int code, const char *msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char *octax_oracle_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ */
/* constants                                                           */
/* ------------------------------------------------------------------ */
/* P:140 "programs loaded at address 0x200"; P:337 font at 0x050-0x09F.  */
#define ROM_BASE 0x200
#define MAX_ROM 3584 /* 4096 - 0x200 */
#define FONT_BASE 0x50
#define W 64
#define H 32

/* Canonical 4x5 hex font (A23).  First byte 0xF0. */
static const uint8_t FONT[80] = {
    0xF0, 0x90, 0x90, 0x90, 0xF0, /* 0 */
    0x20, 0x60, 0x20, 0x20, 0x70, /* 1 */
    0xF0, 0x10, 0xF0, 0x80, 0xF0, /* 2 */
    0xF0, 0x10, 0xF0, 0x10, 0xF0, /* 3 */
    0x90, 0x90, 0xF0, 0x10, 0x10, /* 4 */
    0xF0, 0x80, 0xF0, 0x10, 0xF0, /* 5 */
    0xF0, 0x80, 0xF0, 0x90, 0xF0, /* 6 */
    0xF0, 0x10, 0x20, 0x40, 0x40, /* 7 */
    0xF0, 0x90, 0xF0, 0x90, 0xF0, /* 8 */
    0xF0, 0x90, 0xF0, 0x10, 0xF0, /* 9 */
    0xF0, 0x90, 0xF0, 0x90, 0x90, /* A */
    0xE0, 0x90, 0xE0, 0x90, 0xE0, /* B */
    0xF0, 0x80, 0x80, 0x80, 0xF0, /* C */
    0xE0, 0x90, 0x90, 0x90, 0xE0, /* D */
    0xF0, 0x80, 0xF0, 0x80, 0xF0, /* E */
    0xF0, 0x80, 0xF0, 0x80, 0x80, /* F */
};

/* ------------------------------------------------------------------ */
/* Philox4x32-10 (Random123), used for CXNN (A12) and synthetic        */
/* actions.  Written from the published algorithm definition.          */
/* ------------------------------------------------------------------ */
void octax_oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2],
                                uint32_t out[4]) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; round++) {
    if (round > 0) { /* key schedule: bump between rounds */
      k0 += W0;
      k1 += W1;
    }
    uint64_t p0 = (uint64_t)M0 * (uint64_t)c0;
    uint64_t p1 = (uint64_t)M1 * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0;
    c1 = n1;
    c2 = n2;
    c3 = n3;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

/* A12: CXNN byte = Philox(ctr={draw, episode, gid, 0}, key=seed).out0 & 0xFF */
static uint8_t philox_byte(uint64_t seed, uint64_t gid, uint32_t episode,
                           uint32_t draw) {
  uint32_t ctr[4] = {draw, episode, (uint32_t)gid, 0u};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t out[4];
  octax_oracle_philox4x32_10(ctr, key, out);
  return (uint8_t)(out[0] & 0xFFu);
}

/* SURVEY c.1 "synthetic action": Philox(ctr={t_lo,t_hi,gid,1}, key=aseed) */
int32_t octax_oracle_synthetic_action(uint64_t aseed, uint64_t t, uint64_t gid,
                                      uint32_t n_actions) {
  uint32_t ctr[4] = {(uint32_t)t, (uint32_t)(t >> 32), (uint32_t)gid, 1u};
  uint32_t key[2] = {(uint32_t)aseed, (uint32_t)(aseed >> 32)};
  uint32_t out[4];
  octax_oracle_philox4x32_10(ctr, key, out);
  if (n_actions == 0) return 0;
  return (int32_t)(out[0] % n_actions);
}

/* ------------------------------------------------------------------ */
/* expression language (P:152-154 score_fn / terminated_fn; grammar   */
/* and u32 semantics from S:250-283).  Recursive-descent AST.          */
/* ------------------------------------------------------------------ */
typedef enum {
  N_NUM, N_REG, N_I, N_DT, N_ST, N_MEM, N_NEG, N_NOT, N_BNOT,
  N_MUL, N_DIV, N_MOD, N_ADD, N_SUB, N_SHL, N_SHR,
  N_LT, N_LE, N_GT, N_GE, N_EQ, N_NE, N_BAND, N_BXOR, N_BOR, N_LAND, N_LOR
} node_kind;

typedef struct node {
  node_kind kind;
  uint32_t value; /* N_NUM literal, N_REG index */
  struct node *a, *b;
} node;

typedef struct {
  const char *s;
  size_t pos;
  bool err;
  size_t err_pos;
  char msg[128];
} parser;

static void free_node(node *n) {
  if (!n) return;
  free_node(n->a);
  free_node(n->b);
  free(n);
}

static node *mk(node_kind k, uint32_t v, node *a, node *b) {
  node *n = (node *)calloc(1, sizeof(node));
  if (!n) {
    free_node(a);
    free_node(b);
    return NULL;
  }
  n->kind = k;
  n->value = v;
  n->a = a;
  n->b = b;
  return n;
}

static void perr(parser *p, const char *m) {
  if (!p->err) {
    p->err = true;
    p->err_pos = p->pos;
    snprintf(p->msg, sizeof p->msg, "%s", m);
  }
}

static void skip_ws(parser *p) {
  while (p->s[p->pos] == ' ' || p->s[p->pos] == '\t' || p->s[p->pos] == '\n' ||
         p->s[p->pos] == '\r')
    p->pos++;
}

static bool is_ident_char(char c) {
  return (c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z') ||
         (c >= '0' && c <= '9') || c == '_';
}

static int lower(int c) { return (c >= 'A' && c <= 'Z') ? c + 32 : c; }

/* match a keyword case-insensitively as a whole identifier */
static bool match_word(parser *p, const char *w) {
  size_t n = strlen(w);
  for (size_t i = 0; i < n; i++)
    if (lower((unsigned char)p->s[p->pos + i]) != w[i]) return false;
  if (is_ident_char(p->s[p->pos + n])) return false;
  p->pos += n;
  return true;
}

static bool match_op(parser *p, const char *op) {
  skip_ws(p);
  size_t n = strlen(op);
  if (strncmp(p->s + p->pos, op, n) != 0) return false;
  p->pos += n;
  return true;
}

static bool parse_number(parser *p, uint32_t *out) {
  const char *s = p->s;
  size_t i = p->pos;
  uint64_t v = 0;
  if (s[i] == '0' && (s[i + 1] == 'x' || s[i + 1] == 'X')) {
    i += 2;
    size_t start = i;
    while (1) {
      int c = lower((unsigned char)s[i]);
      int d;
      if (c >= '0' && c <= '9') d = c - '0';
      else if (c >= 'a' && c <= 'f') d = c - 'a' + 10;
      else break;
      v = v * 16 + (uint64_t)d;
      if (v > 0xFFFFFFFFull) { perr(p, "literal out of range"); return false; }
      i++;
    }
    if (i == start) { perr(p, "bad hex literal"); return false; }
  } else if (s[i] >= '0' && s[i] <= '9') {
    while (s[i] >= '0' && s[i] <= '9') {
      v = v * 10 + (uint64_t)(s[i] - '0');
      if (v > 0xFFFFFFFFull) { perr(p, "literal out of range"); return false; }
      i++;
    }
  } else {
    return false;
  }
  if (is_ident_char(s[i])) { p->pos = i; perr(p, "bad literal"); return false; }
  p->pos = i;
  *out = (uint32_t)v;
  return true;
}

static node *parse_expr(parser *p);

static node *parse_primary(parser *p) {
  skip_ws(p);
  const char *s = p->s;
  char c = s[p->pos];
  uint32_t num;
  if (c == '(') {
    p->pos++;
    node *e = parse_expr(p);
    if (p->err) { free_node(e); return NULL; }
    if (!match_op(p, ")")) { free_node(e); perr(p, "expected ')'"); return NULL; }
    return e;
  }
  if (c >= '0' && c <= '9') {
    if (!parse_number(p, &num)) return NULL;
    return mk(N_NUM, num, NULL, NULL);
  }
  /* V0..V15 (decimal), VA..VF (hex letter), V[n] */
  if (lower((unsigned char)c) == 'v') {
    char d = s[p->pos + 1];
    if (d == '[') {
      p->pos += 2;
      skip_ws(p);
      if (!parse_number(p, &num)) { perr(p, "expected register number"); return NULL; }
      if (num > 15) { perr(p, "register index > 15"); return NULL; }
      if (!match_op(p, "]")) { perr(p, "expected ']'"); return NULL; }
      return mk(N_REG, num, NULL, NULL);
    }
    if (d >= '0' && d <= '9') {
      size_t i = p->pos + 1;
      uint32_t v = 0;
      while (s[i] >= '0' && s[i] <= '9') { v = v * 10 + (uint32_t)(s[i] - '0'); i++; if (v > 99) break; }
      if (is_ident_char(s[i]) || v > 15) { perr(p, "bad register name"); return NULL; }
      p->pos = i;
      return mk(N_REG, v, NULL, NULL);
    }
    int l = lower((unsigned char)d);
    if (l >= 'a' && l <= 'f' && !is_ident_char(s[p->pos + 2])) {
      p->pos += 2;
      return mk(N_REG, (uint32_t)(l - 'a' + 10), NULL, NULL);
    }
    perr(p, "bad register name");
    return NULL;
  }
  if (match_word(p, "dt")) return mk(N_DT, 0, NULL, NULL);
  if (match_word(p, "st")) return mk(N_ST, 0, NULL, NULL);
  if (match_word(p, "i")) return mk(N_I, 0, NULL, NULL);
  {
    size_t save = p->pos;
    if (match_word(p, "mem") || match_word(p, "memory")) {
      if (!match_op(p, "[")) { perr(p, "expected '['"); return NULL; }
      node *e = parse_expr(p);
      if (p->err) { free_node(e); return NULL; }
      if (!match_op(p, "]")) { free_node(e); perr(p, "expected ']'"); return NULL; }
      return mk(N_MEM, 0, e, NULL);
    }
    p->pos = save;
  }
  perr(p, c ? "unexpected character" : "unexpected end of expression");
  return NULL;
}

static node *parse_unary(parser *p) {
  skip_ws(p);
  char c = p->s[p->pos];
  if (c == '-' || c == '~' || (c == '!' && p->s[p->pos + 1] != '=')) {
    p->pos++;
    node *a = parse_unary(p);
    if (p->err) { free_node(a); return NULL; }
    return mk(c == '-' ? N_NEG : c == '~' ? N_BNOT : N_NOT, 0, a, NULL);
  }
  return parse_primary(p);
}

/* binary levels, loosest first ("standard precedence") */
typedef struct { const char *tok; node_kind kind; const char *not_followed; } binop;

static node *parse_level(parser *p, int level);

static const binop L_LOR[] = {{"||", N_LOR, NULL}, {NULL, 0, NULL}};
static const binop L_LAND[] = {{"&&", N_LAND, NULL}, {NULL, 0, NULL}};
static const binop L_BOR[] = {{"|", N_BOR, "|"}, {NULL, 0, NULL}};
static const binop L_BXOR[] = {{"^", N_BXOR, NULL}, {NULL, 0, NULL}};
static const binop L_BAND[] = {{"&", N_BAND, "&"}, {NULL, 0, NULL}};
static const binop L_EQ[] = {{"==", N_EQ, NULL}, {"!=", N_NE, NULL}, {NULL, 0, NULL}};
static const binop L_REL[] = {{"<=", N_LE, NULL}, {">=", N_GE, NULL},
                              {"<", N_LT, "<"}, {">", N_GT, ">"}, {NULL, 0, NULL}};
static const binop L_SH[] = {{"<<", N_SHL, NULL}, {">>", N_SHR, NULL}, {NULL, 0, NULL}};
static const binop L_ADD[] = {{"+", N_ADD, NULL}, {"-", N_SUB, NULL}, {NULL, 0, NULL}};
static const binop L_MUL[] = {{"*", N_MUL, NULL}, {"//", N_DIV, NULL},
                              {"/", N_DIV, NULL}, {"%", N_MOD, NULL}, {NULL, 0, NULL}};
static const binop *LEVELS[] = {L_LOR, L_LAND, L_BOR, L_BXOR, L_BAND,
                                L_EQ,  L_REL,  L_SH,  L_ADD,  L_MUL};
#define N_LEVELS 10

static node *parse_level(parser *p, int level) {
  if (level == N_LEVELS) return parse_unary(p);
  node *lhs = parse_level(p, level + 1);
  if (p->err) { free_node(lhs); return NULL; }
  for (;;) {
    skip_ws(p);
    const binop *hit = NULL;
    for (const binop *b = LEVELS[level]; b->tok; b++) {
      size_t n = strlen(b->tok);
      if (strncmp(p->s + p->pos, b->tok, n) != 0) continue;
      if (b->not_followed && strncmp(p->s + p->pos + n, b->not_followed,
                                     strlen(b->not_followed)) == 0)
        continue;
      hit = b;
      break;
    }
    if (!hit) return lhs;
    p->pos += strlen(hit->tok);
    node *rhs = parse_level(p, level + 1);
    if (p->err) { free_node(lhs); free_node(rhs); return NULL; }
    lhs = mk(hit->kind, 0, lhs, rhs);
    if (!lhs) { perr(p, "out of memory"); return NULL; }
  }
}

static node *parse_expr(parser *p) { return parse_level(p, 0); }

static node *parse_full(const char *s, size_t *err_pos, char *msg, size_t msg_len) {
  parser p;
  memset(&p, 0, sizeof p);
  p.s = s;
  node *e = parse_expr(&p);
  if (!p.err) {
    skip_ws(&p);
    if (p.s[p.pos] != '\0') perr(&p, "unexpected trailing input");
  }
  if (p.err) {
    free_node(e);
    if (err_pos) *err_pos = p.err_pos;
    if (msg) snprintf(msg, msg_len, "%s at byte %zu", p.msg, p.err_pos);
    return NULL;
  }
  return e;
}

/* ------------------------------------------------------------------ */
/* one CHIP-8 machine + RL bookkeeping       */
/* ------------------------------------------------------------------ */
typedef struct {
  uint8_t mem[4096];
  uint8_t V[16];
  uint16_t I, PC;
  uint8_t SP;
  uint16_t stk[16];
  uint8_t DT, ST;
  bool disp[H][W];
  bool halted;
  uint16_t keys;
  uint32_t episode, draw, steps, prev_score;
  int32_t ep_ret;
  bool hist[4][H][W]; /* oldest .. newest; hist[3] == disp between steps */
  bool fr[4][H][W];   /* OBS_STACK_FRAMES: displays after the last 4 frames of the step */
  uint64_t gid;
  uint64_t cls_count[16]; /* workload trace: cycles by op>>12 */
  uint64_t rows_drawn;
} vm;

struct oracle_env {
  uint8_t rom[MAX_ROM];
  size_t rom_len;
  uint32_t frame_skip, ipf, max_steps, quirks, obs_format;
  uint8_t action_keys[16];
  uint32_t n_action_keys;
  oracle_startup_seg *startup;
  uint32_t n_startup;
  node *score, *term;
  uint64_t n, seed, env_offset;
  int64_t stats[4]; /* sum_returns, episodes, env_steps, error_flags */
  vm *vms;
};

/* eval(expr) : u32 wrap arithmetic, x/0 = x%0 = 0, logic -> 0/1 */
static uint32_t eval_node(const node *n, const vm *m) {
  uint32_t a, b;
  switch (n->kind) {
  case N_NUM: return n->value;
  case N_REG: return m->V[n->value];
  case N_I: return m->I;
  case N_DT: return m->DT;
  case N_ST: return m->ST;
  case N_MEM: return m->mem[eval_node(n->a, m) & 0xFFFu];
  case N_NEG: return 0u - eval_node(n->a, m);
  case N_NOT: return eval_node(n->a, m) == 0u ? 1u : 0u;
  case N_BNOT: return ~eval_node(n->a, m);
  default: break;
  }
  a = eval_node(n->a, m);
  b = eval_node(n->b, m);
  switch (n->kind) {
  case N_MUL: return a * b;
  case N_DIV: return b == 0u ? 0u : a / b;
  case N_MOD: return b == 0u ? 0u : a % b;
  case N_ADD: return a + b;
  case N_SUB: return a - b;
  case N_SHL: return b >= 32u ? 0u : a << b; /* reading A27 */
  case N_SHR: return b >= 32u ? 0u : a >> b;
  case N_LT: return a < b;
  case N_LE: return a <= b;
  case N_GT: return a > b;
  case N_GE: return a >= b;
  case N_EQ: return a == b;
  case N_NE: return a != b;
  case N_BAND: return a & b;
  case N_BXOR: return a ^ b;
  case N_BOR: return a | b;
  case N_LAND: return (a != 0u && b != 0u) ? 1u : 0u;
  case N_LOR: return (a != 0u || b != 0u) ? 1u : 0u;
  default: return 0u;
  }
}

/* power_on(j): mem := 0; font at 0x50; rom at 0x200; registers 0; PC := 0x200 */
static void power_on(const oracle_env *e, vm *m) {
  memset(m->mem, 0, sizeof m->mem);
  memcpy(m->mem + FONT_BASE, FONT, sizeof FONT);
  memcpy(m->mem + ROM_BASE, e->rom, e->rom_len);
  memset(m->V, 0, sizeof m->V);
  m->I = 0;
  m->SP = 0;
  memset(m->stk, 0, sizeof m->stk);
  m->DT = 0;
  m->ST = 0;
  m->PC = ROM_BASE;
  memset(m->disp, 0, sizeof m->disp);
  m->halted = false;
  m->keys = 0;
  m->draw = 0;
}

/* draw_sprite: P:144 (XOR render), P:327/P:333 (collision when a pixel
   turns off); clipping and address rules A18, A21. */
static void draw_sprite(const oracle_env *e, vm *m, int x, int y, int n) {
  int x0 = m->V[x] & 63;
  int y0 = m->V[y] & 31;
  bool hit = false;
  int base = m->I & 0xFFF;
  bool wrap = (e->quirks & ORACLE_Q_WRAP_SPRITES) != 0;
  for (int r = 0; r < n; r++) {
    int yy = y0 + r;
    if (yy >= H) {
      if (wrap) yy &= 31;
      else break;
    }
    int a = base + r;
    uint8_t byte = a <= 0xFFF ? m->mem[a] : 0;
    m->rows_drawn++;
    for (int c = 0; c < 8; c++) {
      if (!((byte >> (7 - c)) & 1)) continue;
      int xx = x0 + c;
      if (xx >= W) {
        if (wrap) xx &= 63;
        else continue;
      }
      if (m->disp[yy][xx]) hit = true;
      m->disp[yy][xx] = !m->disp[yy][xx];
    }
  }
  m->V[0xF] = hit ? 1 : 0;
}

/* cycle(j): fetch, decode, execute */
static void cycle(const oracle_env *e, vm *m) {
  if (m->PC > 0xFFE) { /* A17 */
    m->halted = true;
    return;
  }
  uint16_t op = (uint16_t)((m->mem[m->PC] << 8) | m->mem[m->PC + 1]);
  m->PC = (uint16_t)(m->PC + 2);
  int x = (op >> 8) & 0xF, y = (op >> 4) & 0xF, n = op & 0xF;
  uint8_t nn = (uint8_t)(op & 0xFF);
  uint16_t nnn = (uint16_t)(op & 0xFFF);
  m->cls_count[op >> 12]++;
  switch (op >> 12) {
  case 0x0:
    if (op == 0x00E0) {
      memset(m->disp, 0, sizeof m->disp);
    } else if (op == 0x00EE) {
      if (m->SP == 0) { m->halted = true; return; }
      m->SP--;
      m->PC = m->stk[m->SP];
    }
    /* else 0NNN: no-op (A20) */
    break;
  case 0x1: m->PC = nnn; break;
  case 0x2:
    if (m->SP == 16) { m->halted = true; return; }
    m->stk[m->SP] = m->PC;
    m->SP++;
    m->PC = nnn;
    break;
  case 0x3: if (m->V[x] == nn) m->PC = (uint16_t)(m->PC + 2); break;
  case 0x4: if (m->V[x] != nn) m->PC = (uint16_t)(m->PC + 2); break;
  case 0x5:
    if (n != 0) { m->halted = true; return; }
    if (m->V[x] == m->V[y]) m->PC = (uint16_t)(m->PC + 2);
    break;
  case 0x6: m->V[x] = nn; break;
  case 0x7: m->V[x] = (uint8_t)(m->V[x] + nn); break; /* VF untouched */
  case 0x8: {
    /* read both operands first; VF written LAST (A15) */
    uint8_t a = m->V[x], b = m->V[y];
    bool vy_shift = (e->quirks & ORACLE_Q_SHIFT_VY) != 0;
    bool vf_reset = (e->quirks & ORACLE_Q_VF_RESET) != 0;
    switch (n) {
    case 0x0: m->V[x] = b; break;
    case 0x1: m->V[x] = a | b; if (vf_reset) m->V[0xF] = 0; break;
    case 0x2: m->V[x] = a & b; if (vf_reset) m->V[0xF] = 0; break;
    case 0x3: m->V[x] = a ^ b; if (vf_reset) m->V[0xF] = 0; break;
    case 0x4: {
      unsigned sum = (unsigned)a + (unsigned)b;
      m->V[x] = (uint8_t)(sum & 0xFF);
      m->V[0xF] = (uint8_t)(sum >> 8);
      break;
    }
    case 0x5:
      m->V[x] = (uint8_t)(a - b);
      m->V[0xF] = a >= b ? 1 : 0;
      break;
    case 0x6: {
      uint8_t s = vy_shift ? b : a;
      m->V[x] = (uint8_t)(s >> 1);
      m->V[0xF] = s & 1;
      break;
    }
    case 0x7:
      m->V[x] = (uint8_t)(b - a);
      m->V[0xF] = b >= a ? 1 : 0;
      break;
    case 0xE: {
      uint8_t s = vy_shift ? b : a;
      m->V[x] = (uint8_t)(s << 1);
      m->V[0xF] = (s >> 7) & 1;
      break;
    }
    default: m->halted = true; return; /* A20 */
    }
    break;
  }
  case 0x9:
    if (n != 0) { m->halted = true; return; }
    if (m->V[x] != m->V[y]) m->PC = (uint16_t)(m->PC + 2);
    break;
  case 0xA: m->I = nnn; break;
  case 0xB: {
    int r = (e->quirks & ORACLE_Q_JUMP_VX) ? x : 0;
    m->PC = (uint16_t)((nnn + m->V[r]) & 0xFFF);
    break;
  }
  case 0xC:
    m->V[x] = philox_byte(e->seed, m->gid, m->episode, m->draw) & nn;
    m->draw++;
    break;
  case 0xD: draw_sprite(e, m, x, y, n); break;
  case 0xE: {
    int k = m->V[x] & 0xF; /* A19 */
    bool down = ((m->keys >> k) & 1) != 0;
    if (nn == 0x9E) { if (down) m->PC = (uint16_t)(m->PC + 2); }
    else if (nn == 0xA1) { if (!down) m->PC = (uint16_t)(m->PC + 2); }
    else { m->halted = true; return; }
    break;
  }
  case 0xF:
    switch (nn) {
    case 0x07: m->V[x] = m->DT; break;
    case 0x0A: /* A16: level-triggered wait */
      if (m->keys != 0) {
        int k = 0;
        while (!((m->keys >> k) & 1)) k++;
        m->V[x] = (uint8_t)k;
      } else {
        m->PC = (uint16_t)(m->PC - 2);
      }
      break;
    case 0x15: m->DT = m->V[x]; break;
    case 0x18: m->ST = m->V[x]; break;
    case 0x1E: m->I = (uint16_t)(m->I + m->V[x]); break; /* 16-bit, no VF */
    case 0x29: m->I = (uint16_t)(FONT_BASE + 5 * (m->V[x] & 0xF)); break;
    case 0x33: /* BCD */
      m->mem[(m->I + 0) & 0xFFF] = (uint8_t)(m->V[x] / 100);
      m->mem[(m->I + 1) & 0xFFF] = (uint8_t)((m->V[x] / 10) % 10);
      m->mem[(m->I + 2) & 0xFFF] = (uint8_t)(m->V[x] % 10);
      break;
    case 0x55:
      for (int k = 0; k <= x; k++) m->mem[(m->I + k) & 0xFFF] = m->V[k];
      if (e->quirks & ORACLE_Q_LOADSTORE_INC_I) m->I = (uint16_t)(m->I + x + 1);
      break;
    case 0x65:
      for (int k = 0; k <= x; k++) m->V[k] = m->mem[(m->I + k) & 0xFFF];
      if (e->quirks & ORACLE_Q_LOADSTORE_INC_I) m->I = (uint16_t)(m->I + x + 1);
      break;
    default: m->halted = true; return;
    }
    break;
  }
}

/* frame(j): ipf cycles then the 60 Hz timer tick (A1, A2) */
static void frame(const oracle_env *e, vm *m) {
  for (uint32_t k = 0; k < e->ipf; k++)
    if (!m->halted) cycle(e, m);
  if (!m->halted) {
    if (m->DT > 0) m->DT--;
    if (m->ST > 0) m->ST--;
  }
}

/* reset(j): power-on, startup segments (A11), bookkeeping */
static void env_reset_one(const oracle_env *e, vm *m) {
  power_on(e, m);
  for (uint32_t s = 0; s < e->n_startup; s++) {
    m->keys = e->startup[s].keymask;
    for (uint32_t f = 0; f < e->startup[s].frames; f++) frame(e, m);
  }
  m->keys = 0;
  m->steps = 0;
  m->prev_score = eval_node(e->score, m);
  for (int p = 0; p < 4; p++) memcpy(m->hist[p], m->disp, sizeof m->disp);
  for (int p = 0; p < 4; p++) memcpy(m->fr[p], m->disp, sizeof m->disp);
  m->ep_ret = 0;
}

static void write_obs(const oracle_env *e, const vm *m, uint8_t *obs_env) {
  /* A3 default: the last 4 step-end displays; OBS_STACK_FRAMES: the last 4 frames */
  const bool(*src)[H][W] = (e->obs_format & ORACLE_OBS_STACK_FRAMES) ? m->fr : m->hist;
  if ((e->obs_format & 1u) == ORACLE_OBS_PACKED) {
    /* obs[p][y][b] = sum_c hist[p][y][8b+c] << (7-c) */
    for (int p = 0; p < 4; p++)
      for (int y = 0; y < H; y++)
        for (int b = 0; b < 8; b++) {
          uint8_t v = 0;
          for (int c = 0; c < 8; c++)
            if (src[p][y][8 * b + c]) v |= (uint8_t)(1u << (7 - c));
          obs_env[(p * H + y) * 8 + b] = v;
        }
  } else {
    /* obs[p][x][y] = hist[p][y][x]  ("(4, 64, 32)"; A4) */
    for (int p = 0; p < 4; p++)
      for (int x = 0; x < W; x++)
        for (int y = 0; y < H; y++)
          obs_env[(p * W + x) * H + y] = src[p][y][x] ? 1 : 0;
  }
}

static size_t obs_bytes(const oracle_env *e) {
  return (e->obs_format & 1u) == ORACLE_OBS_PACKED ? 4u * 32u * 8u : 4u * 64u * 32u;
}

/* ------------------------------------------------------------------ */
/* public API                                                          */
/* ------------------------------------------------------------------ */
static void env_free(oracle_env *e) {
  if (!e) return;
  free_node(e->score);
  free_node(e->term);
  free(e->startup);
  free(e->vms);
  free(e);
}

int octax_oracle_create(const uint8_t *rom, size_t rom_len,
                        const oracle_game_spec *spec, uint64_t n_envs,
                        uint64_t seed, uint64_t env_offset, oracle_env **out) {
  if (!out) return fail(ORACLE_E_INVALID_ARG, "out is NULL");
  *out = NULL;
  if (!spec) return fail(ORACLE_E_INVALID_ARG, "spec is NULL");
  if (rom_len == 0 || !rom) return fail(ORACLE_E_ROM_EMPTY, "ROM is empty");
  if (rom_len > MAX_ROM) return fail(ORACLE_E_ROM_TOO_LARGE, "ROM larger than 3584 bytes");
  if (spec->abi_version != 1) return fail(ORACLE_E_SPEC, "abi_version must be 1");
  if (n_envs == 0) return fail(ORACLE_E_INVALID_ARG, "n_envs must be > 0");
  if (spec->frame_skip == 0) return fail(ORACLE_E_SPEC, "frame_skip must be > 0");
  if (spec->instructions_per_frame == 0) return fail(ORACLE_E_SPEC, "instructions_per_frame must be > 0");
  if (spec->n_action_keys < 1 || spec->n_action_keys > 16 || !spec->action_keys)
    return fail(ORACLE_E_SPEC, "n_action_keys must be in 1..16");
  for (uint32_t i = 0; i < spec->n_action_keys; i++) {
    if (spec->action_keys[i] > 15) return fail(ORACLE_E_SPEC, "action key > 15");
    for (uint32_t j = 0; j < i; j++)
      if (spec->action_keys[j] == spec->action_keys[i])
        return fail(ORACLE_E_SPEC, "duplicate action key");
  }
  if (spec->n_startup > 0 && !spec->startup) return fail(ORACLE_E_SPEC, "startup is NULL");
  if (spec->quirks & ~31u) return fail(ORACLE_E_SPEC, "unknown quirk bits");
  if (spec->obs_format & ~(1u | ORACLE_OBS_STACK_FRAMES)) return fail(ORACLE_E_SPEC, "unknown obs_format");
  if (!spec->score_expr || !spec->terminated_expr)
    return fail(ORACLE_E_SPEC, "expressions must be non-NULL");

  oracle_env *e = (oracle_env *)calloc(1, sizeof(oracle_env));
  if (!e) return fail(ORACLE_E_OOM, "out of memory");
  char msg[200];
  size_t epos = 0;
  e->score = parse_full(spec->score_expr, &epos, msg, sizeof msg);
  if (!e->score) {
    env_free(e);
    char m2[260];
    snprintf(m2, sizeof m2, "score_expr: %s", msg);
    return fail(ORACLE_E_EXPR, m2);
  }
  e->term = parse_full(spec->terminated_expr, &epos, msg, sizeof msg);
  if (!e->term) {
    env_free(e);
    char m2[260];
    snprintf(m2, sizeof m2, "terminated_expr: %s", msg);
    return fail(ORACLE_E_EXPR, m2);
  }
  memcpy(e->rom, rom, rom_len);
  e->rom_len = rom_len;
  e->frame_skip = spec->frame_skip;
  e->ipf = spec->instructions_per_frame;
  e->max_steps = spec->max_episode_steps;
  e->quirks = spec->quirks;
  e->obs_format = spec->obs_format;
  memcpy(e->action_keys, spec->action_keys, spec->n_action_keys);
  e->n_action_keys = spec->n_action_keys;
  e->n_startup = spec->n_startup;
  if (spec->n_startup) {
    e->startup = (oracle_startup_seg *)malloc(sizeof(oracle_startup_seg) * spec->n_startup);
    if (!e->startup) { env_free(e); return fail(ORACLE_E_OOM, "out of memory"); }
    memcpy(e->startup, spec->startup, sizeof(oracle_startup_seg) * spec->n_startup);
  }
  e->n = n_envs;
  e->env_offset = env_offset;
  e->vms = (vm *)calloc((size_t)n_envs, sizeof(vm));
  if (!e->vms) { env_free(e); return fail(ORACLE_E_OOM, "out of memory"); }
  int rc = octax_oracle_reset(e, seed, NULL);
  if (rc != ORACLE_OK) { env_free(e); return rc; }
  *out = e;
  return ORACLE_OK;
}

/* octax_reset(seed): batch seed := seed; for all j: episode := 0; reset(j) */
int octax_oracle_reset(oracle_env *e, uint64_t seed, uint8_t *obs_out) {
  if (!e) return fail(ORACLE_E_INVALID_ARG, "env is NULL");
  e->seed = seed;
  memset(e->stats, 0, sizeof e->stats);
  for (uint64_t j = 0; j < e->n; j++) {
    vm *m = &e->vms[j];
    m->gid = e->env_offset + j; /* A13: RNG keyed by global env id */
    m->episode = 0;
    env_reset_one(e, m);
    if (obs_out) write_obs(e, m, obs_out + j * obs_bytes(e));
  }
  return ORACLE_OK;
}

/* step(j, a): SURVEY c.1 "step" -- P:146, A5-A10, A25.
   Optional extras: final_obs_out (the obs of the terminal transition, written for
   done envs only), episode_return_out / episode_length_out (0 where not done). */
int octax_oracle_step_ex(oracle_env *e, const int32_t *actions, uint8_t *obs_out,
                         float *reward_out, uint8_t *done_out,
                         uint8_t *terminated_out, uint8_t *truncated_out,
                         uint8_t *final_obs_out, int32_t *episode_return_out,
                         uint32_t *episode_length_out) {
  if (!e || !actions) return fail(ORACLE_E_INVALID_ARG, "NULL argument");
  for (uint64_t j = 0; j < e->n; j++) {
    vm *m = &e->vms[j];
    memset(m->cls_count, 0, sizeof m->cls_count);
    m->rows_drawn = 0;
    int32_t a = actions[j];
    if (a < 0 || (uint32_t)a > e->n_action_keys) { /* out of range: no-op + sticky flag */
      e->stats[3] |= 1;
      a = 0;
    }
    m->keys = a == 0 ? 0 : (uint16_t)(1u << e->action_keys[a - 1]); /* A5 */
    for (int p = 0; p < 4; p++) memcpy(m->fr[p], m->disp, sizeof m->disp);
    for (uint32_t f = 0; f < e->frame_skip; f++) {
      frame(e, m);
      /* frame f is plane f + 4 - frame_skip of the intra-step stack (when >= 0) */
      long pl = (long)f + 4 - (long)e->frame_skip;
      if (pl >= 0) memcpy(m->fr[pl], m->disp, sizeof m->disp);
    }
    uint32_t s = eval_node(e->score, m);
    int32_t d = (int32_t)(s - m->prev_score); /* A6, A7: signed delta */
    float reward = (float)d;
    m->prev_score = s;
    m->ep_ret = (int32_t)((uint32_t)m->ep_ret + (uint32_t)d);
    m->steps++;
    bool term = eval_node(e->term, m) != 0u || m->halted; /* A17, A25 */
    bool trunc = e->max_steps > 0 && m->steps >= e->max_steps; /* A9 */
    memmove(m->hist[0], m->hist[1], sizeof m->hist[0]);
    memmove(m->hist[1], m->hist[2], sizeof m->hist[0]);
    memmove(m->hist[2], m->hist[3], sizeof m->hist[0]);
    memcpy(m->hist[3], m->disp, sizeof m->disp);
    e->stats[2] += 1;
    if (episode_return_out) episode_return_out[j] = (term || trunc) ? m->ep_ret : 0;
    if (episode_length_out) episode_length_out[j] = (term || trunc) ? m->steps : 0u;
    if (term || trunc) { /* A10: same-step auto-reset, Gymnax convention */
      if (final_obs_out) write_obs(e, m, final_obs_out + j * obs_bytes(e));
      e->stats[0] += m->ep_ret;
      e->stats[1] += 1;
      m->episode++;
      env_reset_one(e, m);
    }
    if (obs_out) write_obs(e, m, obs_out + j * obs_bytes(e));
    if (reward_out) reward_out[j] = reward;
    if (done_out) done_out[j] = (term || trunc) ? 1 : 0;
    if (terminated_out) terminated_out[j] = term ? 1 : 0;
    if (truncated_out) truncated_out[j] = trunc ? 1 : 0;
  }
  return ORACLE_OK;
}

int octax_oracle_step(oracle_env *e, const int32_t *actions, uint8_t *obs_out,
                      float *reward_out, uint8_t *done_out,
                      uint8_t *terminated_out, uint8_t *truncated_out) {
  return octax_oracle_step_ex(e, actions, obs_out, reward_out, done_out, terminated_out,
                              truncated_out, NULL, NULL, NULL);
}

int octax_oracle_stats(oracle_env *e, int64_t out4[4]) {
  if (!e || !out4) return fail(ORACLE_E_INVALID_ARG, "NULL argument");
  for (int i = 0; i < 4; i++) out4[i] = e->stats[i];
  if (e->stats[3] != 0) return fail(ORACLE_E_DEVICE, "out-of-range action seen");
  return ORACLE_OK;
}

/* canonical per-env state, SURVEY c.6 (5,200 bytes, little-endian) */
static void put16(uint8_t *p, uint16_t v) { p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); }
static void put32(uint8_t *p, uint32_t v) {
  for (int i = 0; i < 4; i++) p[i] = (uint8_t)(v >> (8 * i));
}
static uint16_t get16(const uint8_t *p) { return (uint16_t)(p[0] | (p[1] << 8)); }
static uint32_t get32(const uint8_t *p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

static void pack_display(const bool d[H][W], uint8_t *out256) {
  for (int y = 0; y < H; y++)
    for (int b = 0; b < 8; b++) {
      uint8_t v = 0;
      for (int c = 0; c < 8; c++)
        if (d[y][8 * b + c]) v |= (uint8_t)(1u << (7 - c));
      out256[y * 8 + b] = v;
    }
}

static void unpack_display(const uint8_t *in256, bool d[H][W]) {
  for (int y = 0; y < H; y++)
    for (int x = 0; x < W; x++) d[y][x] = ((in256[y * 8 + x / 8] >> (7 - x % 8)) & 1) != 0;
}

static void vm_to_canon(const vm *m, uint8_t *c) {
  memset(c, 0, ORACLE_CANON_BYTES);
  memcpy(c + 0, m->V, 16);
  put16(c + 16, m->I);
  put16(c + 18, m->PC);
  c[20] = m->SP;
  c[21] = m->DT;
  c[22] = m->ST;
  c[23] = m->halted ? 1 : 0;
  for (int k = 0; k < 16; k++) put16(c + 24 + 2 * k, m->stk[k]);
  put32(c + 56, m->draw);
  put32(c + 60, m->episode);
  put32(c + 64, m->steps);
  put32(c + 68, m->prev_score);
  put32(c + 72, (uint32_t)m->ep_ret);
  pack_display(m->disp, c + 80);
  for (int p = 0; p < 3; p++) pack_display(m->hist[p], c + 336 + 256 * p);
  memcpy(c + 1104, m->mem, 4096);
}

static void canon_to_vm(const uint8_t *c, vm *m) {
  memcpy(m->V, c + 0, 16);
  m->I = get16(c + 16);
  m->PC = get16(c + 18);
  m->SP = c[20];
  m->DT = c[21];
  m->ST = c[22];
  m->halted = (c[23] & 1) != 0;
  for (int k = 0; k < 16; k++) m->stk[k] = get16(c + 24 + 2 * k);
  m->draw = get32(c + 56);
  m->episode = get32(c + 60);
  m->steps = get32(c + 64);
  m->prev_score = get32(c + 68);
  m->ep_ret = (int32_t)get32(c + 72);
  unpack_display(c + 80, m->disp);
  for (int p = 0; p < 3; p++) unpack_display(c + 336 + 256 * p, m->hist[p]);
  memcpy(m->hist[3], m->disp, sizeof m->disp);
  memcpy(m->mem, c + 1104, 4096);
}

int octax_oracle_get_state(oracle_env *e, uint64_t env, uint8_t *canon_out) {
  if (!e || !canon_out) return fail(ORACLE_E_INVALID_ARG, "NULL argument");
  if (env >= e->n) return fail(ORACLE_E_INVALID_ARG, "env index out of range");
  vm_to_canon(&e->vms[env], canon_out);
  return ORACLE_OK;
}

int octax_oracle_set_state(oracle_env *e, uint64_t env, const uint8_t *canon_in) {
  if (!e || !canon_in) return fail(ORACLE_E_INVALID_ARG, "NULL argument");
  if (env >= e->n) return fail(ORACLE_E_INVALID_ARG, "env index out of range");
  if (canon_in[20] > 16) return fail(ORACLE_E_INVALID_ARG, "SP > 16");
  canon_to_vm(canon_in, &e->vms[env]);
  return ORACLE_OK;
}

void octax_oracle_destroy(oracle_env *e) { env_free(e); }

int octax_oracle_run_cycles(oracle_env *e, uint64_t env, uint32_t n, uint16_t keys) {
  if (!e || env >= e->n) return fail(ORACLE_E_INVALID_ARG, "bad env");
  vm *m = &e->vms[env];
  m->keys = keys;
  for (uint32_t k = 0; k < n; k++)
    if (!m->halted) cycle(e, m);
  m->keys = 0;
  return ORACLE_OK;
}

int octax_oracle_run_frames(oracle_env *e, uint64_t env, uint32_t n, uint16_t keys) {
  if (!e || env >= e->n) return fail(ORACLE_E_INVALID_ARG, "bad env");
  vm *m = &e->vms[env];
  m->keys = keys;
  for (uint32_t k = 0; k < n; k++) frame(e, m);
  m->keys = 0;
  return ORACLE_OK;
}

int octax_oracle_tick_timers(oracle_env *e, uint64_t env) {
  if (!e || env >= e->n) return fail(ORACLE_E_INVALID_ARG, "bad env");
  vm *m = &e->vms[env];
  if (!m->halted) {
    if (m->DT > 0) m->DT--;
    if (m->ST > 0) m->ST--;
  }
  return ORACLE_OK;
}

int octax_oracle_eval_expr(const char *expr, const uint8_t *canon_state,
                           uint32_t *value_out, size_t *err_offset_out) {
  if (!expr) return fail(ORACLE_E_INVALID_ARG, "expr is NULL");
  char msg[200];
  size_t epos = 0;
  node *n = parse_full(expr, &epos, msg, sizeof msg);
  if (!n) {
    if (err_offset_out) *err_offset_out = epos;
    return fail(ORACLE_E_EXPR, msg);
  }
  vm *m = (vm *)calloc(1, sizeof(vm));
  if (!m) { free_node(n); return fail(ORACLE_E_OOM, "out of memory"); }
  if (canon_state) canon_to_vm(canon_state, m);
  if (value_out) *value_out = eval_node(n, m);
  free(m);
  free_node(n);
  return ORACLE_OK;
}

int octax_oracle_counters(oracle_env *e, uint64_t env, uint64_t out17[17]) {
  if (!e || env >= e->n || !out17) return fail(ORACLE_E_INVALID_ARG, "bad env");
  for (int i = 0; i < 16; i++) out17[i] = e->vms[env].cls_count[i];
  out17[16] = e->vms[env].rows_drawn;
  return ORACLE_OK;
}
