/* polycert_port.c — plain-C CPU restatement of the reference verifier's
 * widened-double (WidenedFloat64) analysis path.
 *
 * ORACLE / TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load this library, and only as a checker or
 * CPU timing baseline; the product (paper_2007_10868_b200) never links or
 * calls it. Pinned against the compiled reference (oracle/_ref, see
 * tests/test_oracle.py) and the reference's golden vectors
 * (proj/docs/golden/report.jsonl, committed as tests/golden/).
 *
 * Every function follows one reference function; file:line citations are to
 * /root/reference/proj/include/polycert/ headers unless noted. Loop orders, zero
 * skips and the outward-step rounding rule are restated exactly, so results
 * are bit-identical to the reference (compile with -ffp-contract=off).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { K_INPUT = 0, K_DENSE = 1, K_CONV = 2, K_RELU = 3, K_JOIN = 4 };

typedef struct {
  double lo, hi;
} iv;

/* ---------------- numeric core: interval.hpp:38-103 ---------------- */
static const double kResidualFloor = 0x1p-500; /* interval.hpp:48 */

static double step_down(double x) { return nextafter(x, -INFINITY); }
static double step_up(double x) { return nextafter(x, INFINITY); }

static int sum_exact(double a, double b, double s) { /* interval.hpp:50-57 */
  if (!isfinite(s)) return 0;
  double a1 = s - b, b1 = s - a1, da = a - a1, db = b - b1;
  return da + db == 0.0;
}
static double add_down(double a, double b) { /* :59-63 */
  double s = a + b;
  if (isnan(s)) return -INFINITY;
  return sum_exact(a, b, s) ? s : step_down(s);
}
static double add_up(double a, double b) { /* :64-68 */
  double s = a + b;
  if (isnan(s)) return INFINITY;
  return sum_exact(a, b, s) ? s : step_up(s);
}
static int mul_exact(double a, double b, double p) { /* :71-73 */
  return isfinite(p) && fabs(p) >= kResidualFloor && fma(a, b, -p) == 0.0;
}
static double mul_down(double a, double b) { /* :74-78 */
  if (a == 0.0 || b == 0.0) return 0.0;
  double p = a * b;
  return mul_exact(a, b, p) ? p : step_down(p);
}
static double mul_up(double a, double b) { /* :79-83 */
  if (a == 0.0 || b == 0.0) return 0.0;
  double p = a * b;
  return mul_exact(a, b, p) ? p : step_up(p);
}
static int div_exact(double a, double b, double q) { /* :84-86 */
  return isfinite(q) && fabs(a) >= kResidualFloor && fma(q, b, -a) == 0.0;
}
static double div_down(double a, double b) { /* :87-91 */
  if (a == 0.0) return 0.0;
  double q = a / b;
  return div_exact(a, b, q) ? q : step_down(q);
}
static double div_up(double a, double b) { /* :92-96 */
  if (a == 0.0) return 0.0;
  double q = a / b;
  return div_exact(a, b, q) ? q : step_up(q);
}
static double ulp_above(double x) { /* :98-102 */
  double m = fabs(x);
  if (!isfinite(m)) return INFINITY;
  return step_up(m) - m;
}

/* std::max / std::min semantics (first argument wins ties and NaN). */
static double smax(double a, double b) { return (a < b) ? b : a; }
static double smin(double a, double b) { return (b < a) ? b : a; }

static int iv_is_zero(iv a) { return a.lo == 0.0 && a.hi == 0.0; } /* :150 */
static iv ivp(double v) { iv r = {v, v}; return r; }
static iv ivz(void) { iv r = {0.0, 0.0}; return r; }
static iv iv_add(iv a, iv b) { iv r = {add_down(a.lo, b.lo), add_up(a.hi, b.hi)}; return r; } /* :163-170 */
static iv iv_neg(iv a) { iv r = {-a.hi, -a.lo}; return r; }
static iv iv_sub(iv a, iv b) { return iv_add(a, iv_neg(b)); }
static void iv_acc(iv* a, iv b) { /* :185-195 */
  if (iv_is_zero(b)) return;
  a->lo = add_down(a->lo, b.lo);
  a->hi = add_up(a->hi, b.hi);
}
static iv iv_mul_scalar(iv a, double w) { /* :197-208 */
  if (w == 0.0 || iv_is_zero(a)) return ivz();
  iv r;
  if (w > 0.0) { r.lo = mul_down(a.lo, w); r.hi = mul_up(a.hi, w); }
  else { r.lo = mul_down(a.hi, w); r.hi = mul_up(a.lo, w); }
  return r;
}
static iv iv_mul(iv a, iv b) { /* :210-226 */
  if (iv_is_zero(a) || iv_is_zero(b)) return ivz();
  double l1 = mul_down(a.lo, b.lo), l2 = mul_down(a.lo, b.hi);
  double l3 = mul_down(a.hi, b.lo), l4 = mul_down(a.hi, b.hi);
  double u1 = mul_up(a.lo, b.lo), u2 = mul_up(a.lo, b.hi);
  double u3 = mul_up(a.hi, b.lo), u4 = mul_up(a.hi, b.hi);
  iv r = {smin(smin(l1, l2), smin(l3, l4)), smax(smax(u1, u2), smax(u3, u4))};
  return r;
}
static iv iv_div(iv a, iv b) { /* :230-247 (divisor > 0 by construction) */
  if (iv_is_zero(a)) return ivz();
  double l1 = div_down(a.lo, b.lo), l2 = div_down(a.lo, b.hi);
  double l3 = div_down(a.hi, b.lo), l4 = div_down(a.hi, b.hi);
  double u1 = div_up(a.lo, b.lo), u2 = div_up(a.lo, b.hi);
  double u3 = div_up(a.hi, b.lo), u4 = div_up(a.hi, b.hi);
  iv r = {smin(smin(l1, l2), smin(l3, l4)), smax(smax(u1, u2), smax(u3, u4))};
  return r;
}
static iv iv_pos_part(iv a) { iv r = {smax(a.lo, 0.0), smax(a.hi, 0.0)}; return r; } /* :252-256 */
static iv iv_neg_part(iv a) { iv r = {smin(a.lo, 0.0), smin(a.hi, 0.0)}; return r; } /* :258-262 */
static double mag(iv a) { return smax(fabs(a.lo), fabs(a.hi)); }                    /* :264-267 */

/* ---------------- network: network.hpp:84-148 ---------------- */
typedef struct {
  int kind, pred0, pred1;
  int in_w, in_h, in_c, out_w, out_h, out_c;
  int fw, fh, sw, sh, pw, ph, cin, cout;
  int head;
  const double* w; /* dense [out][in] or filter ((fy*fw+fx)*cin+ci)*cout+co */
  const double* b;
} layer_t;

typedef struct {
  int n;
  layer_t* L;
} net_t;

static int numel_out(const layer_t* l) { return l->out_w * l->out_h * l->out_c; }
static int numel_in(const layer_t* l) { return l->in_w * l->in_h * l->in_c; }
static int fidx(int W, int C, int w, int h, int c) { return (h * W + w) * C + c; } /* network.hpp:25 */
static double filt(const layer_t* l, int fx, int fy, int ci, int co) {              /* :145-148 */
  return l->w[((fy * l->fw + fx) * l->cin + ci) * l->cout + co];
}

/* join_head: deepest common ancestor (model_io.cpp:137-160). */
static int join_head(const net_t* net, int j) {
  int n = net->n, best = -1;
  char* aa = calloc((size_t)n, 1);
  char* ab = calloc((size_t)n, 1);
  int* st = malloc(sizeof(int) * (size_t)(2 * n + 2));
  for (int side = 0; side < 2; ++side) {
    char* a = side ? ab : aa;
    int sp = 0;
    st[sp++] = side ? net->L[j].pred1 : net->L[j].pred0;
    while (sp) {
      int x = st[--sp];
      if (a[x]) continue;
      a[x] = 1;
      if (net->L[x].kind == K_INPUT) continue;
      st[sp++] = net->L[x].pred0;
      if (net->L[x].kind == K_JOIN) st[sp++] = net->L[x].pred1;
    }
  }
  for (int x = 0; x < n; ++x)
    if (aa[x] && ab[x] && x > best) best = x;
  free(aa); free(ab); free(st);
  return best;
}

/* ---------------- forward intervals: eval.hpp:109-237 ---------------- */
static iv affine_bound(const iv* xs, const double* ws, int n, int stride_w, double bias, int pad) {
  /* eval.hpp:109-156 (widened branch); ws read with stride (filter columns) */
  double lo = bias, hi = bias, abs_hi = fabs(bias);
  long long terms = 1;
  for (int i = 0; i < n; ++i) {
    double w = ws[(size_t)i * stride_w];
    if (w == 0.0) continue;
    if (pad) {
      ++terms;
      double m = smax(fabs(xs[i].lo), fabs(xs[i].hi));
      abs_hi = add_up(abs_hi, mul_up(fabs(w), m));
    }
    if (w > 0.0) { lo = add_down(lo, mul_down(w, xs[i].lo)); hi = add_up(hi, mul_up(w, xs[i].hi)); }
    else { lo = add_down(lo, mul_down(w, xs[i].hi)); hi = add_up(hi, mul_up(w, xs[i].lo)); }
  }
  if (pad) {
    double slack = 2.0 * (double)(terms + 1) * ulp_above(abs_hi);
    iv r = {add_down(lo, -slack), add_up(hi, slack)};
    return r;
  }
  iv r = {lo, hi};
  return r;
}

static void compute_layer_bounds(const net_t* net, int k, iv** bounds, int pad) { /* eval.hpp:161-228 */
  const layer_t* L = &net->L[k];
  const iv* x = bounds[L->pred0];
  iv* y = bounds[k];
  switch (L->kind) {
    case K_DENSE: {
      int n_out = numel_out(L), n_in = numel_in(L);
      for (int j = 0; j < n_out; ++j) y[j] = affine_bound(x, L->w + (size_t)j * n_in, n_in, 1, L->b[j], pad);
      break;
    }
    case K_CONV: {
      int maxn = L->fw * L->fh * L->cin;
      iv* cs = malloc(sizeof(iv) * (size_t)maxn);
      double* ws = malloc(sizeof(double) * (size_t)maxn);
      for (int h = 0; h < L->out_h; ++h)
        for (int w = 0; w < L->out_w; ++w)
          for (int d = 0; d < L->out_c; ++d) {
            int n = 0;
            for (int fy = 0; fy < L->fh; ++fy) {
              long long iy = (long long)h * L->sh - L->ph + fy;
              if (iy < 0 || iy >= L->in_h) continue;
              for (int fx = 0; fx < L->fw; ++fx) {
                long long ix = (long long)w * L->sw - L->pw + fx;
                if (ix < 0 || ix >= L->in_w) continue;
                for (int ci = 0; ci < L->cin; ++ci) {
                  cs[n] = x[fidx(L->in_w, L->in_c, (int)ix, (int)iy, ci)];
                  ws[n] = filt(L, fx, fy, ci, d);
                  ++n;
                }
              }
            }
            y[fidx(L->out_w, L->out_c, w, h, d)] = affine_bound(cs, ws, n, 1, L->b[d], pad);
          }
      free(cs); free(ws);
      break;
    }
    case K_RELU: {
      int n = numel_out(L);
      for (int i = 0; i < n; ++i) {
        iv r = {x[i].lo > 0.0 ? x[i].lo : 0.0, x[i].hi > 0.0 ? x[i].hi : 0.0};
        y[i] = r;
      }
      break;
    }
    case K_JOIN: {
      const iv* b = bounds[L->pred1];
      int n = numel_out(L);
      for (int i = 0; i < n; ++i) y[i] = iv_add(x[i], b[i]);
      break;
    }
  }
}

/* ---------------- relaxation + dev: analyzer.hpp:23-159 ---------------- */
typedef struct {
  iv alpha, beta, gamma, delta;
} relax_t; /* backsub.hpp:61-64 */

static relax_t relu_relaxation(iv b) { /* analyzer.hpp:38-70 */
  relax_t r;
  iv one = ivp(1.0), zero = ivz();
  if (!(b.lo < 0.0)) { r.alpha = one; r.beta = zero; r.gamma = one; r.delta = zero; }
  else if (!(b.hi > 0.0)) { r.alpha = zero; r.beta = zero; r.gamma = zero; r.delta = zero; }
  else {
    iv den = iv_sub(ivp(b.hi), ivp(b.lo));
    r.gamma = iv_div(ivp(b.hi), den);
    iv num = iv_mul(ivp(-b.lo), ivp(b.hi));
    r.delta = iv_div(num, den);
    r.alpha = b.hi > -b.lo ? one : zero;
    r.beta = zero;
  }
  return r;
}

typedef struct {
  const net_t* net;
  iv** bounds;
  iv** raw;
  relax_t** relax;
  double** dev; /* NULL entry: empty (relu/input) */
  char* feeds_relu;
} state_t;

static void recompute_dev(state_t* st, int from) { /* analyzer.hpp:82-159 */
  const net_t* net = st->net;
  for (int k = from < 1 ? 1 : from; k < net->n; ++k) {
    const layer_t* L = &net->L[k];
    double* dv = st->dev[k];
    switch (L->kind) {
      case K_DENSE: {
        int n_out = numel_out(L), n_in = numel_in(L);
        const iv* x = st->bounds[L->pred0];
        for (int j = 0; j < n_out; ++j) {
          double absrow = fabs(L->b[j]);
          const double* w = L->w + (size_t)j * n_in;
          for (int t = 0; t < n_in; ++t) absrow = add_up(absrow, mul_up(fabs(w[t]), mag(x[t])));
          dv[j] = 2.0 * (double)(n_in + 2) * ulp_above(absrow);
        }
        break;
      }
      case K_CONV: {
        const iv* x = st->bounds[L->pred0];
        for (int h = 0; h < L->out_h; ++h)
          for (int w = 0; w < L->out_w; ++w)
            for (int d = 0; d < L->out_c; ++d) {
              double absrow = fabs(L->b[d]);
              long long terms = 1;
              for (int fy = 0; fy < L->fh; ++fy) {
                long long iy = (long long)h * L->sh - L->ph + fy;
                if (iy < 0 || iy >= L->in_h) continue;
                for (int fx = 0; fx < L->fw; ++fx) {
                  long long ix = (long long)w * L->sw - L->pw + fx;
                  if (ix < 0 || ix >= L->in_w) continue;
                  for (int ci = 0; ci < L->cin; ++ci) {
                    absrow = add_up(absrow, mul_up(fabs(filt(L, fx, fy, ci, d)),
                                                   mag(x[fidx(L->in_w, L->in_c, (int)ix, (int)iy, ci)])));
                    ++terms;
                  }
                }
              }
              dv[fidx(L->out_w, L->out_c, w, h, d)] = 2.0 * (double)(terms + 1) * ulp_above(absrow);
            }
        break;
      }
      case K_JOIN: {
        const iv* a = st->bounds[L->pred0];
        const iv* b = st->bounds[L->pred1];
        int n = numel_out(L);
        for (int j = 0; j < n; ++j) dv[j] = 2.0 * ulp_above(add_up(mag(a[j]), mag(b[j])));
        break;
      }
      default:
        break;
    }
  }
}

/* ---------------- bound matrices: backsub.hpp:85-143 ---------------- */
typedef struct {
  int layer, dense, ww, wh;
  long long* origins; /* rows x 2 (cuboid only) */
} frame_t;

typedef struct {
  int upper; /* Polarity */
  int query_layer;
  frame_t f;
  int row_cells, rows;
  iv* coeff;
  iv* k;
  iv* kraw;
  int* row_index;
} bm_t;

typedef struct {
  long long rows_total, rows_terminated_early, gbc_madds, gbc_dense_equiv, dense_madds, checkpoints;
} stats_t;

static int frame_cells(const frame_t* f, const layer_t* l) {
  return f->dense ? numel_out(l) : f->ww * f->wh * l->out_c;
}

static void bm_free(bm_t* m) {
  free(m->f.origins); free(m->coeff); free(m->k); free(m->kraw); free(m->row_index);
  memset(m, 0, sizeof(*m));
}

static void bm_copy(bm_t* dst, const bm_t* src) {
  *dst = *src;
  size_t nr = (size_t)src->rows;
  dst->coeff = malloc(sizeof(iv) * nr * (size_t)src->row_cells + 1);
  memcpy(dst->coeff, src->coeff, sizeof(iv) * nr * (size_t)src->row_cells);
  dst->k = malloc(sizeof(iv) * nr + 1); memcpy(dst->k, src->k, sizeof(iv) * nr);
  dst->kraw = malloc(sizeof(iv) * nr + 1); memcpy(dst->kraw, src->kraw, sizeof(iv) * nr);
  dst->row_index = malloc(sizeof(int) * nr + 1); memcpy(dst->row_index, src->row_index, sizeof(int) * nr);
  dst->f.origins = NULL;
  if (src->f.origins) {
    dst->f.origins = malloc(sizeof(long long) * 2 * nr + 1);
    memcpy(dst->f.origins, src->f.origins, sizeof(long long) * 2 * nr);
  }
}

static void widen_constant(iv* k, double dev) { /* backsub.hpp:175-179 */
  if (dev == 0.0) return;
  k->lo = add_down(k->lo, -dev);
  k->hi = add_up(k->hi, dev);
}
static void dev_add(double* total, iv c, double dev_j) { /* backsub.hpp:187-193 */
  if (dev_j == 0.0) return;
  *total = add_up(*total, mul_up(mag(c), dev_j));
}

/* init_affine_rows: backsub.hpp:205-268 */
static void init_affine_rows(const state_t* st, int layer, const int* sel, int n_rows, int upper, bm_t* m) {
  const layer_t* L = &st->net->L[layer];
  const double* dev = st->dev[layer];
  memset(m, 0, sizeof(*m));
  m->upper = upper; m->query_layer = layer; m->rows = n_rows;
  m->row_index = malloc(sizeof(int) * (size_t)n_rows + 1);
  memcpy(m->row_index, sel, sizeof(int) * (size_t)n_rows);
  m->f.layer = L->pred0;
  m->k = malloc(sizeof(iv) * (size_t)n_rows + 1);
  m->kraw = malloc(sizeof(iv) * (size_t)n_rows + 1);
  if (L->kind == K_DENSE) {
    int n_in = numel_in(L);
    m->f.dense = 1;
    m->row_cells = n_in;
    m->coeff = calloc((size_t)n_rows * (size_t)n_in + 1, sizeof(iv));
    for (int r = 0; r < n_rows; ++r) {
      int q = sel[r];
      for (int t = 0; t < n_in; ++t) m->coeff[(size_t)r * n_in + t] = ivp(L->w[(size_t)q * n_in + t]);
      iv k = ivp(L->b[q]);
      m->kraw[r] = k;
      if (dev) widen_constant(&k, dev[q]);
      m->k[r] = k;
    }
  } else {
    m->f.dense = 0; m->f.ww = L->fw; m->f.wh = L->fh;
    m->f.origins = malloc(sizeof(long long) * 2 * (size_t)n_rows + 1);
    m->row_cells = L->fw * L->fh * L->in_c;
    m->coeff = calloc((size_t)n_rows * (size_t)m->row_cells + 1, sizeof(iv));
    for (int r = 0; r < n_rows; ++r) {
      int q = sel[r];
      int c = q % L->out_c, w = (q / L->out_c) % L->out_w, h = q / (L->out_c * L->out_w);
      m->f.origins[2 * r] = (long long)w * L->sw - L->pw;
      m->f.origins[2 * r + 1] = (long long)h * L->sh - L->ph;
      iv* row = m->coeff + (size_t)r * m->row_cells;
      for (int fy = 0; fy < L->fh; ++fy)
        for (int fx = 0; fx < L->fw; ++fx)
          for (int ci = 0; ci < L->cin; ++ci) row[(fy * L->fw + fx) * L->in_c + ci] = ivp(filt(L, fx, fy, ci, c));
      iv k = ivp(L->b[c]);
      m->kraw[r] = k;
      if (dev) widen_constant(&k, dev[q]);
      m->k[r] = k;
    }
  }
}

/* init_identity_rows: backsub.hpp:273-310 */
static void init_identity_rows(const state_t* st, int layer, const int* sel, int n_rows, int upper, bm_t* m) {
  const layer_t* L = &st->net->L[layer];
  memset(m, 0, sizeof(*m));
  m->upper = upper; m->query_layer = layer; m->rows = n_rows;
  m->row_index = malloc(sizeof(int) * (size_t)n_rows + 1);
  memcpy(m->row_index, sel, sizeof(int) * (size_t)n_rows);
  m->f.layer = layer;
  if (L->out_w == 1 && L->out_h == 1) {
    m->f.dense = 1;
    m->row_cells = numel_out(L);
    m->coeff = calloc((size_t)n_rows * (size_t)m->row_cells + 1, sizeof(iv));
    for (int r = 0; r < n_rows; ++r) m->coeff[(size_t)r * m->row_cells + sel[r]] = ivp(1.0);
  } else {
    m->f.dense = 0; m->f.ww = 1; m->f.wh = 1;
    m->f.origins = malloc(sizeof(long long) * 2 * (size_t)n_rows + 1);
    m->row_cells = L->out_c;
    m->coeff = calloc((size_t)n_rows * (size_t)m->row_cells + 1, sizeof(iv));
    for (int r = 0; r < n_rows; ++r) {
      int q = sel[r];
      int c = q % L->out_c, w = (q / L->out_c) % L->out_w, h = q / (L->out_c * L->out_w);
      m->f.origins[2 * r] = w; m->f.origins[2 * r + 1] = h;
      m->coeff[(size_t)r * m->row_cells + c] = ivp(1.0);
    }
  }
  m->k = calloc((size_t)n_rows + 1, sizeof(iv));
  m->kraw = calloc((size_t)n_rows + 1, sizeof(iv));
}

/* init_margin_rows: backsub.hpp:314-336 */
static void init_margin_rows(const state_t* st, int label, bm_t* m) {
  const net_t* net = st->net;
  int out = net->n - 1, n = numel_out(&net->L[out]);
  memset(m, 0, sizeof(*m));
  m->upper = 0; m->query_layer = out; m->f.layer = out; m->f.dense = 1; m->row_cells = n;
  m->rows = n - 1;
  m->row_index = malloc(sizeof(int) * (size_t)n);
  m->coeff = calloc((size_t)n * (size_t)n, sizeof(iv));
  m->k = calloc((size_t)n, sizeof(iv));
  m->kraw = calloc((size_t)n, sizeof(iv));
  int r = 0;
  for (int j = 0; j < n; ++j) {
    if (j == label) continue;
    m->row_index[r] = j;
    m->coeff[(size_t)r * n + label] = ivp(1.0);
    m->coeff[(size_t)r * n + j] = ivp(-1.0);
    ++r;
  }
}

/* cuboid cell -> absolute flat index, -1 if dead (e.g. backsub.hpp:372-378) */
static int cell_abs(const bm_t* m, const layer_t* fl, int r, int cell) {
  if (m->f.dense) return cell;
  int C = fl->out_c;
  int cc = cell % C, cw = (cell / C) % m->f.ww, ch = cell / (C * m->f.ww);
  long long aw = m->f.origins[2 * r] + cw, ah = m->f.origins[2 * r + 1] + ch;
  if (aw < 0 || aw >= fl->out_w || ah < 0 || ah >= fl->out_h) return -1;
  return fidx(fl->out_w, C, (int)aw, (int)ah, cc);
}

/* dense_step: backsub.hpp:343-399 */
static void dense_step(const state_t* st, bm_t* m, stats_t* stats) {
  const layer_t* L = &st->net->L[m->f.layer];
  int n_in = numel_in(L);
  const double* dev = st->dev[m->f.layer];
  iv* nc = calloc((size_t)m->rows * (size_t)n_in + 1, sizeof(iv));
  for (int r = 0; r < m->rows; ++r) {
    const iv* row = m->coeff + (size_t)r * m->row_cells;
    iv* nrow = nc + (size_t)r * n_in;
    double dtot = 0.0;
    for (int cell = 0; cell < m->row_cells; ++cell) {
      iv c = row[cell];
      if (iv_is_zero(c)) continue;
      int j = cell_abs(m, L, r, cell);
      if (j < 0) continue;
      iv bt = iv_mul_scalar(c, L->b[j]);
      iv_acc(&m->k[r], bt);
      iv_acc(&m->kraw[r], bt);
      if (dev) dev_add(&dtot, c, dev[j]);
      const double* wrow = L->w + (size_t)j * n_in;
      for (int t = 0; t < n_in; ++t) iv_acc(&nrow[t], iv_mul_scalar(c, wrow[t]));
      stats->dense_madds += n_in;
    }
    if (dev) widen_constant(&m->k[r], dtot);
  }
  free(m->coeff);
  m->coeff = nc;
  m->row_cells = n_in;
  m->f.layer = L->pred0;
  m->f.dense = 1; m->f.ww = m->f.wh = 0;
  free(m->f.origins); m->f.origins = NULL;
}

static int grow_width(int width, int f, int s) { return (width - 1) * s + f; }              /* depsets.hpp:27 */
static long long step_origin(long long o, int s, int p) { return o * (long long)s - p; } /* depsets.hpp:32-34 */

/* gbc_step: backsub.hpp:401-499 */
static void gbc_step(const state_t* st, bm_t* m, stats_t* stats) {
  const layer_t* L = &st->net->L[m->f.layer];
  const double* dev = st->dev[m->f.layer];
  frame_t nf;
  memset(&nf, 0, sizeof(nf));
  nf.layer = L->pred0;
  nf.dense = m->f.dense;
  int n_cells;
  if (nf.dense) n_cells = numel_in(L);
  else {
    nf.ww = grow_width(m->f.ww, L->fw, L->sw);
    nf.wh = grow_width(m->f.wh, L->fh, L->sh);
    nf.origins = malloc(sizeof(long long) * 2 * (size_t)m->rows + 1);
    n_cells = nf.ww * nf.wh * L->in_c;
  }
  iv* nc = calloc((size_t)m->rows * (size_t)n_cells + 1, sizeof(iv));
  for (int r = 0; r < m->rows; ++r) {
    const iv* row = m->coeff + (size_t)r * m->row_cells;
    iv* nrow = nc + (size_t)r * n_cells;
    double dtot = 0.0;
    long long ow = 0, oh = 0;
    if (!m->f.dense) {
      ow = m->f.origins[2 * r]; oh = m->f.origins[2 * r + 1];
      nf.origins[2 * r] = step_origin(ow, L->sw, L->pw);
      nf.origins[2 * r + 1] = step_origin(oh, L->sh, L->ph);
    }
    int cw_n = m->f.dense ? L->out_w : m->f.ww;
    int ch_n = m->f.dense ? L->out_h : m->f.wh;
    for (int ch = 0; ch < ch_n; ++ch)
      for (int cw = 0; cw < cw_n; ++cw) {
        long long aw = m->f.dense ? cw : ow + cw;
        long long ah = m->f.dense ? ch : oh + ch;
        if (aw < 0 || aw >= L->out_w || ah < 0 || ah >= L->out_h) continue;
        for (int d = 0; d < L->out_c; ++d) {
          iv c = row[m->f.dense ? fidx(L->out_w, L->out_c, (int)aw, (int)ah, d)
                                : (ch * m->f.ww + cw) * L->out_c + d];
          if (iv_is_zero(c)) continue;
          iv bt = iv_mul_scalar(c, L->b[d]);
          iv_acc(&m->k[r], bt);
          iv_acc(&m->kraw[r], bt);
          if (dev) dev_add(&dtot, c, dev[fidx(L->out_w, L->out_c, (int)aw, (int)ah, d)]);
          for (int fy = 0; fy < L->fh; ++fy) {
            long long iy = ah * L->sh - L->ph + fy;
            if (iy < 0 || iy >= L->in_h) continue;
            for (int fx = 0; fx < L->fw; ++fx) {
              long long ix = aw * L->sw - L->pw + fx;
              if (ix < 0 || ix >= L->in_w) continue;
              size_t tb;
              if (nf.dense) tb = (size_t)fidx(L->in_w, L->in_c, (int)ix, (int)iy, 0);
              else {
                long long a = (long long)cw * L->sw + fx, b = (long long)ch * L->sh + fy;
                tb = (size_t)((b * nf.ww + a) * L->in_c);
              }
              for (int ci = 0; ci < L->cin; ++ci) iv_acc(&nrow[tb + ci], iv_mul_scalar(c, filt(L, fx, fy, ci, d)));
              stats->gbc_madds += L->cin;
            }
          }
        }
      }
    if (dev) widen_constant(&m->k[r], dtot);
  }
  stats->gbc_dense_equiv += (long long)m->rows * numel_out(L) * numel_in(L);
  free(m->coeff); free(m->f.origins);
  m->coeff = nc;
  m->row_cells = n_cells;
  m->f = nf;
}

/* relu_step: backsub.hpp:501-568 */
static void relu_step(const state_t* st, bm_t* m) {
  const layer_t* L = &st->net->L[m->f.layer];
  int pred = L->pred0;
  const relax_t* relax = st->relax[pred];
  for (int r = 0; r < m->rows; ++r) {
    iv* row = m->coeff + (size_t)r * m->row_cells;
    for (int cell = 0; cell < m->row_cells; ++cell) {
      iv c = row[cell];
      if (iv_is_zero(c)) continue;
      int j = cell_abs(m, L, r, cell);
      if (j < 0) continue;
      const relax_t* R = &relax[j];
      iv sp = m->upper ? R->gamma : R->alpha, op = m->upper ? R->delta : R->beta;
      iv sn = m->upper ? R->alpha : R->gamma, on = m->upper ? R->beta : R->delta;
      if (!(c.lo < 0.0)) {
        iv off = iv_mul(c, op);
        iv_acc(&m->k[r], off); iv_acc(&m->kraw[r], off);
        row[cell] = iv_mul(c, sp);
      } else if (!(c.hi > 0.0)) {
        iv off = iv_mul(c, on);
        iv_acc(&m->k[r], off); iv_acc(&m->kraw[r], off);
        row[cell] = iv_mul(c, sn);
      } else {
        iv pos = iv_pos_part(c), neg = iv_neg_part(c);
        iv offp = iv_mul(pos, op), offn = iv_mul(neg, on);
        iv_acc(&m->k[r], offp); iv_acc(&m->kraw[r], offp);
        iv_acc(&m->k[r], offn); iv_acc(&m->kraw[r], offn);
        row[cell] = iv_add(iv_mul(pos, sp), iv_mul(neg, sn));
      }
    }
  }
  m->f.layer = pred;
}

/* densify: backsub.hpp:578-608 */
static void densify(const state_t* st, bm_t* m) {
  if (m->f.dense) return;
  const layer_t* L = &st->net->L[m->f.layer];
  int n_cells = numel_out(L);
  iv* nc = calloc((size_t)m->rows * (size_t)n_cells + 1, sizeof(iv));
  for (int r = 0; r < m->rows; ++r) {
    const iv* row = m->coeff + (size_t)r * m->row_cells;
    for (int cell = 0; cell < m->row_cells; ++cell) {
      iv c = row[cell];
      if (iv_is_zero(c)) continue;
      int j = cell_abs(m, L, r, cell);
      if (j < 0) continue;
      nc[(size_t)r * n_cells + j] = c;
    }
  }
  free(m->coeff); free(m->f.origins);
  m->coeff = nc; m->row_cells = n_cells;
  m->f.dense = 1; m->f.ww = m->f.wh = 0; m->f.origins = NULL;
}

/* align_add: backsub.hpp:610-688. Returns -1 on the row-invariance logic_error. */
static int align_add(const state_t* st, bm_t* a, bm_t* b) {
  const layer_t* L = &st->net->L[a->f.layer];
  int C = L->out_c;
  if (a->f.dense || b->f.dense) {
    densify(st, a);
    densify(st, b);
    for (int r = 0; r < a->rows; ++r) {
      iv* ar = a->coeff + (size_t)r * a->row_cells;
      const iv* br = b->coeff + (size_t)r * b->row_cells;
      for (int cell = 0; cell < a->row_cells; ++cell) iv_acc(&ar[cell], br[cell]);
      iv_acc(&a->k[r], b->k[r]);
      iv_acc(&a->kraw[r], b->kraw[r]);
    }
    return 0;
  }
  frame_t nf;
  memset(&nf, 0, sizeof(nf));
  nf.layer = a->f.layer;
  nf.origins = malloc(sizeof(long long) * 2 * (size_t)a->rows + 1);
  long long dw = 0, dh = 0;
  for (int r = 0; r < a->rows; ++r) {
    long long aow = a->f.origins[2 * r], aoh = a->f.origins[2 * r + 1];
    long long bow = b->f.origins[2 * r], boh = b->f.origins[2 * r + 1];
    long long ow = aow < bow ? aow : bow, oh = aoh < boh ? aoh : boh;
    long long ew = aow + a->f.ww > bow + b->f.ww ? aow + a->f.ww : bow + b->f.ww;
    long long eh = aoh + a->f.wh > boh + b->f.wh ? aoh + a->f.wh : boh + b->f.wh;
    nf.origins[2 * r] = ow; nf.origins[2 * r + 1] = oh;
    if (r == 0) { dw = ew - ow; dh = eh - oh; }
    else if (dw != ew - ow || dh != eh - oh) { free(nf.origins); return -1; }
  }
  nf.ww = (int)dw; nf.wh = (int)dh;
  int n_cells = nf.ww * nf.wh * C;
  iv* nc = calloc((size_t)a->rows * (size_t)n_cells + 1, sizeof(iv));
  for (int r = 0; r < a->rows; ++r) {
    iv* nrow = nc + (size_t)r * n_cells;
    for (int side = 0; side < 2; ++side) {
      const bm_t* src = side ? b : a;
      const iv* row = src->coeff + (size_t)r * src->row_cells;
      for (int cell = 0; cell < src->row_cells; ++cell) {
        iv c = row[cell];
        if (iv_is_zero(c)) continue;
        int cc = cell % C, cw = (cell / C) % src->f.ww, chh = cell / (C * src->f.ww);
        long long aw = src->f.origins[2 * r] + cw, ah = src->f.origins[2 * r + 1] + chh;
        long long rw = aw - nf.origins[2 * r], rh = ah - nf.origins[2 * r + 1];
        iv_acc(&nrow[(rh * nf.ww + rw) * C + cc], c);
      }
    }
    iv_acc(&a->k[r], b->k[r]);
    iv_acc(&a->kraw[r], b->kraw[r]);
  }
  free(a->coeff); free(a->f.origins);
  a->coeff = nc; a->row_cells = n_cells; a->f = nf;
  return 0;
}

/* concretize: backsub.hpp:725-764 (+ corner_hi/lo :151-171) */
static void concretize(const state_t* st, iv** fb, const bm_t* m, int raw, double* out) {
  const layer_t* L = &st->net->L[m->f.layer];
  const iv* B = fb[m->f.layer];
  const iv* kc = raw ? m->kraw : m->k;
  for (int r = 0; r < m->rows; ++r) {
    const iv* row = m->coeff + (size_t)r * m->row_cells;
    double acc = m->upper ? kc[r].hi : kc[r].lo;
    for (int cell = 0; cell < m->row_cells; ++cell) {
      iv c = row[cell];
      if (iv_is_zero(c)) continue;
      int j = cell_abs(m, L, r, cell);
      if (j < 0) continue;
      iv b = B[j];
      if (m->upper) {
        double v = mul_up(c.lo, b.lo);
        v = smax(v, mul_up(c.lo, b.hi)); v = smax(v, mul_up(c.hi, b.lo)); v = smax(v, mul_up(c.hi, b.hi));
        acc = add_up(acc, v);
      } else {
        double v = mul_down(c.lo, b.lo);
        v = smin(v, mul_down(c.lo, b.hi)); v = smin(v, mul_down(c.hi, b.lo)); v = smin(v, mul_down(c.hi, b.hi));
        acc = add_down(acc, v);
      }
    }
    out[r] = acc;
  }
}

/* CandidateSet: backsub.hpp:775-818 */
typedef struct {
  double *lo, *hi, *rlo, *rhi;
  char *has_lo, *has_hi, *frozen;
} cand_t;

static int cand_stable(const cand_t* c, int q) {
  if (!c->has_lo[q] || !c->has_hi[q]) return 0;
  return !(c->rlo[q] < 0.0) || !(c->rhi[q] > 0.0);
}

/* compact_rows: backsub.hpp:820-845 */
static void compact_rows(bm_t* m, const char* frozen) {
  int keep = 0;
  for (int r = 0; r < m->rows; ++r) {
    if (frozen[m->row_index[r]]) continue;
    if (keep != r) {
      memmove(m->coeff + (size_t)keep * m->row_cells, m->coeff + (size_t)r * m->row_cells, sizeof(iv) * (size_t)m->row_cells);
      m->k[keep] = m->k[r]; m->kraw[keep] = m->kraw[r];
      m->row_index[keep] = m->row_index[r];
      if (!m->f.dense) { m->f.origins[2 * keep] = m->f.origins[2 * r]; m->f.origins[2 * keep + 1] = m->f.origins[2 * r + 1]; }
    }
    ++keep;
  }
  m->rows = keep;
}

/* walk context: the checkpoint closure of run_backsubstitution / run_margin_pass */
typedef struct {
  const state_t* st;
  iv** raw_bounds;
  bm_t *up, *lo;
  cand_t* cand;
  int allow_freeze, early_term, margin;
  double* best; char* has; /* margin pass */
  stats_t* stats;
  double *vals, *rvals;
} ckpt_t;

static void checkpoint(ckpt_t* c) {
  c->stats->checkpoints++;
  if (c->margin) { /* backsub.hpp:1082-1091 */
    concretize(c->st, c->st->bounds, c->lo, 0, c->vals);
    for (int r = 0; r < c->lo->rows; ++r)
      if (!c->has[r] || c->vals[r] > c->best[r]) { c->best[r] = c->vals[r]; c->has[r] = 1; }
    return;
  }
  cand_t* cd = c->cand; /* backsub.hpp:1032-1054 */
  concretize(c->st, c->st->bounds, c->up, 0, c->vals);
  concretize(c->st, c->raw_bounds, c->up, 1, c->rvals);
  for (int r = 0; r < c->up->rows; ++r) {
    int q = c->up->row_index[r];
    if (cd->frozen[q]) continue;
    if (!cd->has_hi[q] || c->vals[r] < cd->hi[q]) { cd->hi[q] = c->vals[r]; cd->has_hi[q] = 1; }
    if (c->rvals[r] < cd->rhi[q]) cd->rhi[q] = c->rvals[r];
  }
  concretize(c->st, c->st->bounds, c->lo, 0, c->vals);
  concretize(c->st, c->raw_bounds, c->lo, 1, c->rvals);
  for (int r = 0; r < c->lo->rows; ++r) {
    int q = c->lo->row_index[r];
    if (cd->frozen[q]) continue;
    if (!cd->has_lo[q] || c->vals[r] > cd->lo[q]) { cd->lo[q] = c->vals[r]; cd->has_lo[q] = 1; }
    if (c->rvals[r] > cd->rlo[q]) cd->rlo[q] = c->rvals[r];
  }
  if (!c->allow_freeze) return;
  int any = 0;
  for (int r = 0; r < c->up->rows; ++r) {
    int q = c->up->row_index[r];
    if (!cd->frozen[q] && cand_stable(cd, q)) {
      cd->frozen[q] = 1; any = 1;
      if (c->early_term) c->stats->rows_terminated_early++;
    }
  }
  if (c->early_term && any) { compact_rows(c->up, cd->frozen); compact_rows(c->lo, cd->frozen); }
}

static int join_step(const state_t* st, bm_t* m, stats_t* stats);

/* walk_back: backsub.hpp:854-893. ck == NULL: no checkpoints (join branches). */
static int walk_back(const state_t* st, bm_t* up, bm_t* lo, int stop, stats_t* stats, ckpt_t* ck) {
  bm_t* any = up ? up : lo;
  int pending = 0;
  while (any->f.layer != stop) {
    if (any->rows == 0) return 0;
    const layer_t* L = &st->net->L[any->f.layer];
    switch (L->kind) {
      case K_DENSE:
        if (up) dense_step(st, up, stats);
        if (lo) dense_step(st, lo, stats);
        if (ck) checkpoint(ck);
        pending = 0;
        break;
      case K_CONV:
        if (up) gbc_step(st, up, stats);
        if (lo) gbc_step(st, lo, stats);
        if (ck) checkpoint(ck);
        pending = 0;
        break;
      case K_RELU:
        if (up) relu_step(st, up);
        if (lo) relu_step(st, lo);
        pending = 1;
        break;
      case K_JOIN:
        if (up && join_step(st, up, stats)) return -1;
        if (lo && join_step(st, lo, stats)) return -1;
        if (ck) checkpoint(ck);
        pending = 0;
        break;
      default:
        return -2; /* walked through the input layer */
    }
  }
  if (pending && ck) checkpoint(ck);
  return 0;
}

/* join_step: backsub.hpp:694-715 */
static int join_step(const state_t* st, bm_t* m, stats_t* stats) {
  const layer_t* L = &st->net->L[m->f.layer];
  bm_t mb;
  bm_copy(&mb, m);
  memset(mb.k, 0, sizeof(iv) * (size_t)mb.rows);
  memset(mb.kraw, 0, sizeof(iv) * (size_t)mb.rows);
  m->f.layer = L->pred0;
  mb.f.layer = L->pred1;
  int rc = walk_back(st, m->upper ? m : NULL, m->upper ? NULL : m, L->head, stats, NULL);
  if (!rc) rc = walk_back(st, mb.upper ? &mb : NULL, mb.upper ? NULL : &mb, L->head, stats, NULL);
  if (!rc) rc = align_add(st, m, &mb);
  bm_free(&mb);
  return rc;
}

/* chunk sizing: backsub.hpp:904-987 */
typedef struct {
  int dense;
  long long ww, wh;
} sim_t;

static long long sim_cells(const net_t* net, int layer, sim_t s) {
  const layer_t* l = &net->L[layer];
  return s.dense ? numel_out(l) : s.ww * s.wh * l->out_c;
}

static long long sim_walk(const net_t* net, int layer, sim_t* st, int stop) {
  long long peak = sim_cells(net, layer, *st);
  while (layer != stop) {
    const layer_t* L = &net->L[layer];
    switch (L->kind) {
      case K_DENSE: st->dense = 1; st->ww = st->wh = 0; layer = L->pred0; break;
      case K_CONV:
        if (!st->dense) {
          st->ww = grow_width((int)(st->ww < (1 << 20) ? st->ww : (1 << 20)), L->fw, L->sw);
          st->wh = grow_width((int)(st->wh < (1 << 20) ? st->wh : (1 << 20)), L->fh, L->sh);
        }
        layer = L->pred0;
        break;
      case K_RELU: layer = L->pred0; break;
      case K_JOIN: {
        sim_t sa = *st, sb = *st;
        long long pa = sim_walk(net, L->pred0, &sa, L->head);
        long long pb = sim_walk(net, L->pred1, &sb, L->head);
        if (pa + pb > peak) peak = pa + pb;
        layer = L->head;
        if (sa.dense || sb.dense) { st->dense = 1; st->ww = st->wh = 0; }
        else { st->dense = 0; st->ww = sa.ww + sb.ww; st->wh = sa.wh + sb.wh; }
        break;
      }
      default: return peak;
    }
    long long c = sim_cells(net, layer, *st);
    if (c > peak) peak = c;
  }
  return peak;
}

static long long rows_per_chunk(const net_t* net, int q, long long chunk_rows, long long budget) {
  if (chunk_rows > 0) return chunk_rows;
  const layer_t* Q = &net->L[q];
  sim_t s = {1, 0, 0};
  int start = q;
  if (Q->kind == K_CONV) { s.dense = 0; s.ww = Q->fw; s.wh = Q->fh; start = Q->pred0; }
  else if (Q->kind == K_DENSE) start = Q->pred0;
  else if (Q->out_w > 1 || Q->out_h > 1) { s.dense = 0; s.ww = 1; s.wh = 1; }
  long long cells = sim_walk(net, start, &s, 0);
  if (cells < 1) cells = 1;
  long long per_row = cells * 16 * 4 + 1024;
  if (budget < per_row) budget = per_row;
  long long r = budget / per_row;
  return r < 1 ? 1 : r;
}

/* run_backsubstitution: backsub.hpp:993-1065 */
static int run_backsubstitution(state_t* st, int t, int allow_freeze, int early_term, long long chunk_rows,
                                long long budget, stats_t* stats) {
  const net_t* net = st->net;
  const layer_t* Q = &net->L[t];
  int n = numel_out(Q);
  cand_t cd;
  cd.lo = malloc(sizeof(double) * n); cd.hi = malloc(sizeof(double) * n);
  cd.rlo = malloc(sizeof(double) * n); cd.rhi = malloc(sizeof(double) * n);
  cd.has_lo = malloc((size_t)n); cd.has_hi = malloc((size_t)n); cd.frozen = calloc((size_t)n, 1);
  for (int q = 0; q < n; ++q) {
    cd.lo[q] = st->bounds[t][q].lo; cd.hi[q] = st->bounds[t][q].hi;
    cd.rlo[q] = st->raw[t][q].lo; cd.rhi[q] = st->raw[t][q].hi;
    cd.has_lo[q] = cd.has_hi[q] = 1;
  }
  if (allow_freeze)
    for (int q = 0; q < n; ++q)
      if (cand_stable(&cd, q)) { cd.frozen[q] = 1; if (early_term) stats->rows_terminated_early++; }
  stats->rows_total += n;
  int* live = malloc(sizeof(int) * (size_t)n + 1);
  int nlive = 0;
  for (int q = 0; q < n; ++q)
    if (!(early_term && cd.frozen[q])) live[nlive++] = q;
  int affine = Q->kind == K_DENSE || Q->kind == K_CONV;
  long long chunk = rows_per_chunk(net, t, chunk_rows, budget);
  int rc = 0;
  for (long long base = 0; base < nlive && !rc; base += chunk) {
    int cnt = (int)((nlive - base) < chunk ? (nlive - base) : chunk);
    bm_t up, lo;
    if (affine) {
      init_affine_rows(st, t, live + base, cnt, 1, &up);
      init_affine_rows(st, t, live + base, cnt, 0, &lo);
    } else {
      init_identity_rows(st, t, live + base, cnt, 1, &up);
      init_identity_rows(st, t, live + base, cnt, 0, &lo);
    }
    ckpt_t ck;
    memset(&ck, 0, sizeof(ck));
    ck.st = st; ck.raw_bounds = st->raw; ck.up = &up; ck.lo = &lo; ck.cand = &cd;
    ck.allow_freeze = allow_freeze; ck.early_term = early_term; ck.stats = stats;
    ck.vals = malloc(sizeof(double) * (size_t)cnt + 1);
    ck.rvals = malloc(sizeof(double) * (size_t)cnt + 1);
    if (affine) checkpoint(&ck);
    rc = walk_back(st, &up, &lo, 0, stats, &ck);
    free(ck.vals); free(ck.rvals);
    bm_free(&up); bm_free(&lo);
  }
  for (int q = 0; q < n; ++q) {
    st->bounds[t][q].lo = cd.lo[q]; st->bounds[t][q].hi = cd.hi[q];
    st->raw[t][q].lo = cd.rlo[q]; st->raw[t][q].hi = cd.rhi[q];
  }
  free(cd.lo); free(cd.hi); free(cd.rlo); free(cd.rhi); free(cd.has_lo); free(cd.has_hi); free(cd.frozen);
  free(live);
  return rc;
}

/* run_margin_pass: backsub.hpp:1070-1096 */
static int run_margin_pass(state_t* st, int label, double* out, stats_t* stats) {
  bm_t lo;
  init_margin_rows(st, label, &lo);
  int nr = lo.rows;
  stats->rows_total += nr;
  ckpt_t ck;
  memset(&ck, 0, sizeof(ck));
  ck.st = st; ck.lo = &lo; ck.margin = 1; ck.stats = stats;
  ck.best = out;
  ck.has = calloc((size_t)nr + 1, 1);
  ck.vals = malloc(sizeof(double) * (size_t)nr + 1);
  for (int r = 0; r < nr; ++r) out[r] = 0.0;
  int rc = walk_back(st, NULL, &lo, 0, stats, &ck);
  for (int r = 0; r < nr && !rc; ++r)
    if (!ck.has[r]) rc = -3;
  free(ck.has); free(ck.vals);
  bm_free(&lo);
  return rc;
}

/* ---------------- public C ABI ---------------- */

/* input_box: network.hpp:160-177 (widened). Returns -1 if a clamped center is outside [0,1]. */
int port_input_box(const double* center, int n, double eps, int clamp01, double* lo, double* hi) {
  if (eps < 0.0) return -1;
  for (int i = 0; i < n; ++i) {
    double c = center[i];
    double l = add_down(c, -eps), h = add_up(c, eps);
    if (clamp01) {
      if (c < 0.0 || 1.0 < c) return -1;
      l = smax(l, 0.0);
      h = smin(h, 1.0);
    }
    lo[i] = l; hi[i] = h;
  }
  return 0;
}

/* layer_info row (16 ints): kind, n_preds, pred0, pred1, out_w, out_h, out_c,
 * fw, fh, sw, sh, pw, ph, cin, cout, (unused). weights[k]/bias[k] point at
 * the layer's parameters in the reference's flat layouts.
 * label < 0: analysis only. stats[6] mirrors PassStats. Bounds optional.
 * Returns 0, or <0 on an internal error (logic_error analogue). */
int port_analyze(const int* info, int n_layers, const double* const* weights, const double* const* bias,
                 const double* box_lo, const double* box_hi, int label, int early_term, long long chunk_rows,
                 long long memory_budget, int* verified, double* margins, long long* stats_out, double* b_lo,
                 double* b_hi, double* r_lo, double* r_hi) {
  net_t net;
  net.n = n_layers;
  net.L = calloc((size_t)n_layers, sizeof(layer_t));
  for (int k = 0; k < n_layers; ++k) {
    const int* I = info + 16 * k;
    layer_t* l = &net.L[k];
    l->kind = I[0]; l->pred0 = I[2]; l->pred1 = I[3];
    l->out_w = I[4]; l->out_h = I[5]; l->out_c = I[6];
    l->fw = I[7]; l->fh = I[8]; l->sw = I[9]; l->sh = I[10]; l->pw = I[11]; l->ph = I[12];
    l->cin = I[13]; l->cout = I[14];
    l->w = weights ? weights[k] : NULL; l->b = bias ? bias[k] : NULL;
    l->head = -1;
    if (k > 0) {
      const layer_t* p = &net.L[l->pred0];
      l->in_w = p->out_w; l->in_h = p->out_h; l->in_c = p->out_c;
    }
  }
  for (int k = 0; k < n_layers; ++k)
    if (net.L[k].kind == K_JOIN) net.L[k].head = join_head(&net, k);

  state_t st;
  st.net = &net;
  st.bounds = calloc((size_t)n_layers, sizeof(iv*));
  st.raw = calloc((size_t)n_layers, sizeof(iv*));
  st.relax = calloc((size_t)n_layers, sizeof(relax_t*));
  st.dev = calloc((size_t)n_layers, sizeof(double*));
  st.feeds_relu = calloc((size_t)n_layers, 1);
  for (int k = 0; k < n_layers; ++k) {
    int n = numel_out(&net.L[k]);
    st.bounds[k] = calloc((size_t)n + 1, sizeof(iv));
    st.raw[k] = calloc((size_t)n + 1, sizeof(iv));
    if (net.L[k].kind == K_DENSE || net.L[k].kind == K_CONV || net.L[k].kind == K_JOIN)
      st.dev[k] = calloc((size_t)n + 1, sizeof(double));
    if (net.L[k].kind == K_RELU) st.feeds_relu[net.L[k].pred0] = 1;
  }
  /* analyze: analyzer.hpp:198-242 */
  int n0 = numel_out(&net.L[0]);
  for (int i = 0; i < n0; ++i) {
    st.bounds[0][i].lo = box_lo[i]; st.bounds[0][i].hi = box_hi[i];
    st.raw[0][i] = st.bounds[0][i];
  }
  for (int k = 1; k < n_layers; ++k) compute_layer_bounds(&net, k, st.bounds, 1);
  for (int k = 1; k < n_layers; ++k) compute_layer_bounds(&net, k, st.raw, 0);
  for (int k = 0; k < n_layers; ++k)
    if (st.feeds_relu[k]) {
      int n = numel_out(&net.L[k]);
      st.relax[k] = malloc(sizeof(relax_t) * (size_t)n + 1);
      for (int j = 0; j < n; ++j) st.relax[k][j] = relu_relaxation(st.bounds[k][j]);
    }
  recompute_dev(&st, 1);
  stats_t stats;
  memset(&stats, 0, sizeof(stats));
  int out = n_layers - 1, rc = 0;
  for (int t = 1; t < n_layers && !rc; ++t) {
    int is_out = t == out;
    if (!is_out && !st.feeds_relu[t]) continue;
    rc = run_backsubstitution(&st, t, !is_out, early_term, chunk_rows, memory_budget > 0 ? memory_budget : (1ll << 30),
                              &stats);
    if (rc || is_out) continue;
    if (st.feeds_relu[t]) {
      int n = numel_out(&net.L[t]);
      for (int j = 0; j < n; ++j) st.relax[t][j] = relu_relaxation(st.bounds[t][j]);
    }
    for (int k = t + 1; k < n_layers; ++k) {
      compute_layer_bounds(&net, k, st.bounds, 1);
      compute_layer_bounds(&net, k, st.raw, 0);
      if (st.feeds_relu[k]) {
        int n = numel_out(&net.L[k]);
        for (int j = 0; j < n; ++j) st.relax[k][j] = relu_relaxation(st.bounds[k][j]);
      }
    }
    recompute_dev(&st, t + 1);
  }
  if (!rc && label >= 0) { /* verify_robustness: analyzer.hpp:256-276 */
    int n_out = numel_out(&net.L[out]);
    if (label >= n_out) rc = -4;
    else {
      double* lows = malloc(sizeof(double) * (size_t)n_out);
      rc = run_margin_pass(&st, label, lows, &stats);
      int v = 1;
      for (int r = 0; r < n_out - 1; ++r) {
        if (margins) margins[r] = lows[r];
        if (!(lows[r] > 0.0)) v = 0;
      }
      if (verified) *verified = rc ? 0 : v;
      free(lows);
    }
  }
  if (stats_out) {
    stats_out[0] = stats.rows_total; stats_out[1] = stats.rows_terminated_early;
    stats_out[2] = stats.gbc_madds; stats_out[3] = stats.gbc_dense_equiv;
    stats_out[4] = stats.dense_madds; stats_out[5] = stats.checkpoints;
  }
  size_t off = 0;
  for (int k = 0; k < n_layers; ++k) {
    int n = numel_out(&net.L[k]);
    for (int j = 0; j < n; ++j) {
      if (b_lo) b_lo[off + j] = st.bounds[k][j].lo;
      if (b_hi) b_hi[off + j] = st.bounds[k][j].hi;
      if (r_lo) r_lo[off + j] = st.raw[k][j].lo;
      if (r_hi) r_hi[off + j] = st.raw[k][j].hi;
    }
    off += (size_t)n;
  }
  for (int k = 0; k < n_layers; ++k) { free(st.bounds[k]); free(st.raw[k]); free(st.relax[k]); free(st.dev[k]); }
  free(st.bounds); free(st.raw); free(st.relax); free(st.dev); free(st.feeds_relu); free(net.L);
  return rc;
}

/* Scalar ops exported for the numeric-core parity tests (op: 0 add_down,
 * 1 add_up, 2 mul_down, 3 mul_up, 4 div_down, 5 div_up, 6 ulp_above(a)). */
/* Serial chains (test infrastructure): acc0[c] += terms[c*len + j] for j
 * ascending with add_up / add_down, NaN terms skipped (backsub.hpp:740-760). */
void port_chain_fold(int n_chains, int len, const double* acc0, const double* terms, const int* up,
                     double* out) {
  for (int c = 0; c < n_chains; ++c) {
    double acc = acc0[c];
    for (int j = 0; j < len; ++j) {
      const double t = terms[(long long)c * len + j];
      if (t == t) acc = up[c] ? add_up(acc, t) : add_down(acc, t);
    }
    out[c] = acc;
  }
}

void port_scalar_ops(int op, const double* a, const double* b, double* out, long long n) {
  for (long long i = 0; i < n; ++i) {
    switch (op) {
      case 0: out[i] = add_down(a[i], b[i]); break;
      case 1: out[i] = add_up(a[i], b[i]); break;
      case 2: out[i] = mul_down(a[i], b[i]); break;
      case 3: out[i] = mul_up(a[i], b[i]); break;
      case 4: out[i] = div_down(a[i], b[i]); break;
      case 5: out[i] = div_up(a[i], b[i]); break;
      default: out[i] = ulp_above(a[i]); break;
    }
  }
}
