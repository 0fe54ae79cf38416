/*
 * glassnet_oracle.c -- plain, slow, obviously-correct fp64 CPU GlassNet forward pass.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this.  It shares no code,
 * header, table or constant with the CUDA path (paper_2405_19056_b200/csrc).
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, P:n = line n):
 *   1. normalise   x = [G', D], G' = G except pos*2^-3, depth*2^-7; record depth*2^-7
 *                  (reading R9 -- the paper position-encodes all inputs, P:373-375,
 *                  which presumes bounded inputs).  With pe_L > 0
 *                   x and every record are then positionally encoded
 *                  (og_posenc): F0 reads 15(2L+1) channels, h's layer 1 11(2L+1) (+ c0).
 *   2. F (scene encoder): e0 = ReLU(conv3x3_s1(x)), e_l = ReLU(conv3x3_s2(e_{l-1})).
 *   3. T (Eq. eq:SymmetricNN): tau = g(h(b_1),...,h(b_t)) = sum_i h(b_i), h a
 *      shared 2-layer ReLU MLP over each VALID fragment record (k < min(n,K)) -- or, with
 *      sigma_cond (the paper's literal h(b_i, sigma), "sigma is a
 *      scene representation"), over the concatenation [b_i ; sigma], sigma = e0 at the pixel
 *      (the scene encoder's level-0 features, reading N1); the sum is
 *      taken per channel over the values sorted ascending (a pure function of the
 *      multiset -> exactly permutation invariant, table:OrderLoss P:666-679);
 *      tau = [sum, n] (or [sum/n, n] in mean mode, 0 when n = 0).
 *   4. B: phi = ReLU(W_B [e0; tau] + b_B).
 *   5. R: d_{L-1} = e_{L-1}; y_l = ReLU(conv3x3_s1(d_l)) at level l;
 *      d_{l-1} = crop(up2(y_l)) + (l-1 >= 1 ? e_{l-1} : phi); up2 = bilinear,
 *      half-pixel, edge clamp.  Output = sigmoid(W_O [d0; L_d] + b_O) (L_d raw).
 *   Layer widths are BASELINE.json configs[0]/[1] (the paper gives none).
 *
 * Arithmetic: fp64, single thread, direct nested loops, no blocking, no fusion.
 * Every dot product starts from the bias and adds products in index order.
 * Parity pins: tests/test_oracle_pins.py (P1..P14 of SURVEY.md §8(c)).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int H, W, K, L;
  int c[4];
  int h;
  int pool;        /* 0 = sum, 1 = mean                         */
  int r_takes_ld;  /* 1: output 1x1 takes [d0; L_d] (reading R15) */
  int input_norm;  /* 1: power-of-two input normalisation (R9)    */
  int sigma_cond;  /* 1: h(b, sigma), sigma = e0 at the pixel (N1) */
  int pe_L;        /* N2: positional encoding with L_pe frequencies (0 = off)              */
  int objects;     /* N4: object-major buffers, h a 3x3 CNN (og_forward_objects)            */
} og_dims;

typedef struct {        /* optional per-layer dumps (any pointer may be NULL) */
  double* x;            /* [H][W][15]                 */
  double* e[4];         /* level l: [H_l][W_l][c_l]   */
  double* tau;          /* [H][W][h+1]                */
  double* phi;          /* [H][W][c0]                 */
  double* y[4];         /* y_l at level l (l>=1): [H_l][W_l][c_{l-1}] */
  double* d[4];         /* d_l (l = 0..L-2): [H_l][W_l][c_l]          */
  double* logits;       /* [H][W][3]                  */
} og_dump;

static double relu(double v) { return v > 0.0 ? v : 0.0; }

/* N2 -- positional encoding (§3.4 P:373-375 "All the inputs use
 * positional encoding by Mildenhall et al."; the formula as SPEC.md S:395-403 states it):
 *   gamma(v) = (v, sin(2^0 pi v), cos(2^0 pi v), ..., sin(2^(L-1) pi v), cos(2^(L-1) pi v))
 * per channel, channels concatenated in input order: n channels -> n (2L + 1) (DESIGN.md
 * reading N2).  L = 0: the identity. */
void og_posenc(const double* v, int n, int L, double* out) {
  const double pi = 3.14159265358979323846;
  for (int c = 0; c < n; ++c) {
    double* o = out + (size_t)c * (2 * L + 1);
    o[0] = v[c];
    for (int k = 0; k < L; ++k) {
      const double a = ldexp(1.0, k) * pi * v[c];
      o[1 + 2 * k] = sin(a);
      o[2 + 2 * k] = cos(a);
    }
  }
}

static int lvl_size(int n, int l) { /* ceil(n / 2^l) */
  for (int i = 0; i < l; ++i) n = (n + 1) / 2;
  return n;
}

size_t og_weight_count(const og_dims* d) {
  size_t n = 0;
  int h = d->h;
  const int pe = 2 * d->pe_L + 1;          /* N2: channels per encoded input channel */
  const int taps = d->objects ? 9 : 1;     /* N4: h's layers are 3x3 convolutions */
  n += (size_t)h * taps * (11 * pe + (d->sigma_cond ? d->c[0] : 0)) + h;   /* T1 */
  n += (size_t)h * taps * h + h;           /* T2 */
  int cin = 15 * pe;
  for (int l = 0; l < d->L; ++l) { n += (size_t)d->c[l] * 9 * cin + d->c[l]; cin = d->c[l]; }
  n += (size_t)d->c[0] * (d->c[0] + h + 1) + d->c[0];   /* B */
  for (int l = d->L - 1; l >= 1; --l) n += (size_t)d->c[l - 1] * 9 * d->c[l] + d->c[l - 1];
  int nin = d->c[0] + (d->r_takes_ld ? 3 : 0);
  n += (size_t)3 * nin + 3;                /* O */
  return n;
}

/* conv3x3, cross-correlation, OHWI weights, zero padding 1.
 * out[y][x][o] = b[o] + sum_{ky,kx,i} W[o][ky][kx][i] * in[s*y+ky-1][s*x+kx-1][i]. */
void og_conv3x3(const double* in, int H, int W, int Cin, const double* Wt, const double* b,
                int Cout, int stride, int do_relu, double* out) {
  int Ho = (H + stride - 1) / stride, Wo = (W + stride - 1) / stride;
  for (int y = 0; y < Ho; ++y)
    for (int x = 0; x < Wo; ++x)
      for (int o = 0; o < Cout; ++o) {
        double acc = b[o];
        for (int ky = 0; ky < 3; ++ky) {
          int iy = stride * y + ky - 1;
          if (iy < 0 || iy >= H) continue;
          for (int kx = 0; kx < 3; ++kx) {
            int ix = stride * x + kx - 1;
            if (ix < 0 || ix >= W) continue;
            const double* wp = Wt + (((size_t)o * 3 + ky) * 3 + kx) * Cin;
            const double* ip = in + ((size_t)iy * W + ix) * Cin;
            for (int i = 0; i < Cin; ++i) acc += wp[i] * ip[i];
          }
        }
        out[((size_t)y * Wo + x) * Cout + o] = do_relu ? relu(acc) : acc;
      }
}

/* bilinear x2, align_corners=False (half-pixel), edge clamp, cropped to H2 x W2.
 * 1-D: fine[2i] = 0.25 v[max(i-1,0)] + 0.75 v[i]; fine[2i+1] = 0.75 v[i] + 0.25 v[min(i+1,n-1)];
 * 2-D: sum over the 4 taps of (wy * wx) * v (reading R14). */
void og_up2(const double* in, int h, int w, int C, int H2, int W2, double* out) {
  for (int Y = 0; Y < H2; ++Y) {
    int i = Y / 2, ya, yb; double wa, wb;
    if (Y % 2 == 0) { ya = i > 0 ? i - 1 : 0; yb = i; wa = 0.25; wb = 0.75; }
    else            { ya = i; yb = i + 1 < h ? i + 1 : h - 1; wa = 0.75; wb = 0.25; }
    for (int X = 0; X < W2; ++X) {
      int j = X / 2, xa, xb; double va, vb;
      if (X % 2 == 0) { xa = j > 0 ? j - 1 : 0; xb = j; va = 0.25; vb = 0.75; }
      else            { xa = j; xb = j + 1 < w ? j + 1 : w - 1; va = 0.75; vb = 0.25; }
      for (int c = 0; c < C; ++c) {
        double s = (wa * va) * in[((size_t)ya * w + xa) * C + c];
        s += (wa * vb) * in[((size_t)ya * w + xb) * C + c];
        s += (wb * va) * in[((size_t)yb * w + xa) * C + c];
        s += (wb * vb) * in[((size_t)yb * w + xb) * C + c];
        out[((size_t)Y * W2 + X) * C + c] = s;
      }
    }
  }
}

static int cmp_double(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* T for one pixel (Eq. eq:SymmetricNN; readings R2-R7).
 * rec: [K][11] raw records; n: valid count (clamped to K); sigma: [c0] scene features at the
 * pixel (used only with d->sigma_cond: layer 1 then takes [record ; sigma], W1 [h][11 + c0]);
 * tau_out: [h+1]. */
void og_T_pixel(const og_dims* d, const double* W1, const double* b1, const double* W2,
                const double* b2, const double* rec, int n, const double* sigma, double* tau_out) {
  int h = d->h, K = d->K;
  const int pe = 2 * d->pe_L + 1, nr = 11 * pe;          /* N2: encoded record width */
  const int ns = d->sigma_cond ? d->c[0] : 0, nin = nr + ns;
  int m = n < K ? n : K;
  double* a2 = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1) * h);
  double* a1 = (double*)malloc(sizeof(double) * (size_t)h);
  double* col = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
  for (int k = 0; k < m; ++k) {
    double r0[11], r[11 * 21];
    for (int i = 0; i < 11; ++i) r0[i] = rec[(size_t)k * 11 + i];
    if (d->input_norm) r0[7] = r0[7] * 0x1p-7;          /* record depth (R9) */
    og_posenc(r0, 11, d->pe_L, r);                       /* N2 (identity when pe_L = 0) */
    for (int o = 0; o < h; ++o) {                        /* h layer 1 over [gamma(b) ; sigma] */
      double acc = b1[o];
      for (int i = 0; i < nr; ++i) acc += W1[(size_t)o * nin + i] * r[i];
      for (int j = 0; j < ns; ++j) acc += W1[(size_t)o * nin + nr + j] * sigma[j];
      a1[o] = relu(acc);
    }
    for (int o = 0; o < h; ++o) {                        /* h layer 2 */
      double acc = b2[o];
      for (int i = 0; i < h; ++i) acc += W2[(size_t)o * h + i] * a1[i];
      a2[(size_t)k * h + o] = relu(acc);
    }
  }
  for (int j = 0; j < h; ++j) {                          /* g = sum (sorted per channel) */
    for (int k = 0; k < m; ++k) col[k] = a2[(size_t)k * h + j];
    qsort(col, (size_t)m, sizeof(double), cmp_double);
    double s = 0.0;
    for (int k = 0; k < m; ++k) s += col[k];
    if (d->pool == 1) s = m > 0 ? s / (double)m : 0.0;
    tau_out[j] = s;
  }
  tau_out[h] = (double)m;
  free(a2); free(a1); free(col);
}

/* N4 -- object-major transparency buffers with a spatial h (PAPER.md P:257-258
 * "a set of buffers with a size of (w, h, c*(t+1))" -- one full-frame buffer per transparent
 * object; "other networks use multi-layer CNN without down-sampling"; streaming,
 * "the model can operate on a single buffer of each transparent object, and then add
 * it to the summed latent representation").  DESIGN.md reading N4:
 *   x_i   = cover_i ? b_i' : 0        b_i' = b_i with depth x 2^-7 (R9); 11 ch per pixel
 *   a_i   = ReLU(conv3x3(ReLU(conv3x3(x_i; T1)); T2))      h, zero padding, no down-sampling
 *   tau   = [ sum_{i covering the pixel} a_i , n ]      n = number of covering objects
 * (the per-channel sum taken over the values sorted ascending: a function of the multiset of
 * objects, so object order cannot change a bit); B, F, R and the output as og_forward.
 * T1.W [h][3][3][11], T2.W [h][3][3][h] (OHWI) replace the MLP weights in the blob. */
typedef struct {
  int t;                      /* number of objects              */
  const double* const* buf;   /* t x [H][W][11]                 */
  const uint8_t* const* cover;/* t x [H][W], nonzero = covered  */
} og_objects;

static int og_forward_impl(const og_dims* d, const double* wts, const double* gbuf, const double* direct,
                           const double* tbuf, const uint8_t* tcount, const og_objects* ob, double* out,
                           const og_dump* dump) {
  const int H = d->H, W = d->W, K = d->K, L = d->L, h = d->h;
  const int* c = d->c;
  const size_t P = (size_t)H * W;
  if (L < 2 || L > 4 || K < 1 || H < 1 || W < 1 || d->pe_L < 0 || d->pe_L > 10) return 1;
  if ((ob != 0) != (d->objects != 0) || (ob && (d->pe_L || d->sigma_cond))) return 1;
  const int taps = ob ? 9 : 1;
  const int pe = 2 * d->pe_L + 1, nx = 15 * pe;          /* N2: encoded input width */

  /* ---- unpack the weight blob (SURVEY.md §8(b) order) ---- */
  const double* p = wts;
  const double *T1W = p; p += (size_t)h * taps * (11 * pe + (d->sigma_cond ? c[0] : 0)); const double* T1b = p; p += h;
  const double *T2W = p; p += (size_t)h * taps * h;  const double* T2b = p; p += h;
  const double *FW[4], *Fb[4];
  int cin = nx;
  for (int l = 0; l < L; ++l) { FW[l] = p; p += (size_t)c[l] * 9 * cin; Fb[l] = p; p += c[l]; cin = c[l]; }
  const int nB = c[0] + h + 1;
  const double* BW = p; p += (size_t)c[0] * nB; const double* Bb = p; p += c[0];
  const double *RW[4] = {0}, *Rb[4] = {0};
  for (int l = L - 1; l >= 1; --l) { RW[l] = p; p += (size_t)c[l - 1] * 9 * c[l]; Rb[l] = p; p += c[l - 1]; }
  const int nO = c[0] + (d->r_takes_ld ? 3 : 0);
  const double* OW = p; p += (size_t)3 * nO; const double* Ob = p;

  int Hl[4], Wl[4];
  for (int l = 0; l < L; ++l) { Hl[l] = lvl_size(H, l); Wl[l] = lvl_size(W, l); }

  /* ---- 1. normalise (then N2's positional encoding, identity when pe_L = 0) ---- */
  double* x = (double*)malloc(sizeof(double) * P * nx);
  for (size_t q = 0; q < P; ++q) {
    double v[15];
    for (int i = 0; i < 12; ++i) v[i] = gbuf[q * 12 + i];
    for (int i = 0; i < 3; ++i) v[12 + i] = direct[q * 3 + i];
    if (d->input_norm) {
      for (int i = 0; i < 3; ++i) v[i] = v[i] * 0x1p-3;  /* position */
      v[11] = v[11] * 0x1p-7;                            /* depth */
    }
    og_posenc(v, 15, d->pe_L, x + q * nx);
  }
  /* ---- 2. F ---- */
  double* e[4];
  e[0] = (double*)malloc(sizeof(double) * P * c[0]);
  og_conv3x3(x, H, W, nx, FW[0], Fb[0], c[0], 1, 1, e[0]);
  for (int l = 1; l < L; ++l) {
    e[l] = (double*)malloc(sizeof(double) * (size_t)Hl[l] * Wl[l] * c[l]);
    og_conv3x3(e[l - 1], Hl[l - 1], Wl[l - 1], c[l - 1], FW[l], Fb[l], c[l], 2, 1, e[l]);
  }
  /* ---- 3. T ---- */
  double* tau = (double*)malloc(sizeof(double) * P * (h + 1));
  if (!ob) {
    for (size_t q = 0; q < P; ++q)
      og_T_pixel(d, T1W, T1b, T2W, T2b, tbuf + q * (size_t)K * 11, (int)tcount[q], e[0] + q * c[0],
                 tau + q * (h + 1));
  } else {   /* N4: one object buffer at a time through the spatial h */
    const int t = ob->t;
    double* vals = (double*)malloc(sizeof(double) * P * (size_t)(t > 0 ? t : 1) * h);
    int* cnt = (int*)calloc(P, sizeof(int));
    double* xi = (double*)malloc(sizeof(double) * P * 11);
    double* h1 = (double*)malloc(sizeof(double) * P * h);
    double* a2 = (double*)malloc(sizeof(double) * P * h);
    double* col = (double*)malloc(sizeof(double) * (size_t)(t > 0 ? t : 1));
    for (int i = 0; i < t; ++i) {
      for (size_t q = 0; q < P; ++q)
        for (int j = 0; j < 11; ++j) {
          double v = ob->cover[i][q] ? ob->buf[i][q * 11 + j] : 0.0;
          if (j == 7 && d->input_norm) v = v * 0x1p-7;
          xi[q * 11 + j] = v;
        }
      og_conv3x3(xi, H, W, 11, T1W, T1b, h, 1, 1, h1);
      og_conv3x3(h1, H, W, h, T2W, T2b, h, 1, 1, a2);
      for (size_t q = 0; q < P; ++q)
        if (ob->cover[i][q]) {
          for (int j = 0; j < h; ++j) vals[(q * t + cnt[q]) * h + j] = a2[q * h + j];
          cnt[q] += 1;
        }
    }
    for (size_t q = 0; q < P; ++q) {
      const int m = cnt[q];
      for (int j = 0; j < h; ++j) {
        for (int k = 0; k < m; ++k) col[k] = vals[(q * t + k) * h + j];
        qsort(col, (size_t)m, sizeof(double), cmp_double);
        double sm = 0.0;
        for (int k = 0; k < m; ++k) sm += col[k];
        if (d->pool == 1) sm = m > 0 ? sm / (double)m : 0.0;
        tau[q * (h + 1) + j] = sm;
      }
      tau[q * (h + 1) + h] = (double)m;
    }
    free(vals); free(cnt); free(xi); free(h1); free(a2); free(col);
  }
  /* ---- 4. B ---- */
  double* phi = (double*)malloc(sizeof(double) * P * c[0]);
  for (size_t q = 0; q < P; ++q)
    for (int o = 0; o < c[0]; ++o) {
      double acc = Bb[o];
      for (int i = 0; i < c[0]; ++i) acc += BW[(size_t)o * nB + i] * e[0][q * c[0] + i];
      for (int i = 0; i <= h; ++i) acc += BW[(size_t)o * nB + c[0] + i] * tau[q * (h + 1) + i];
      phi[q * c[0] + o] = relu(acc);
    }
  /* ---- 5. R ---- */
  double* dl = e[L - 1];                 /* d_{L-1} = e_{L-1} (borrowed) */
  double* dbuf[4] = {0};
  double* ybuf[4] = {0};
  for (int l = L - 1; l >= 1; --l) {
    ybuf[l] = (double*)malloc(sizeof(double) * (size_t)Hl[l] * Wl[l] * c[l - 1]);
    og_conv3x3(dl, Hl[l], Wl[l], c[l], RW[l], Rb[l], c[l - 1], 1, 1, ybuf[l]);
    size_t n = (size_t)Hl[l - 1] * Wl[l - 1] * c[l - 1];
    dbuf[l - 1] = (double*)malloc(sizeof(double) * n);
    og_up2(ybuf[l], Hl[l], Wl[l], c[l - 1], Hl[l - 1], Wl[l - 1], dbuf[l - 1]);
    const double* skip = (l - 1 >= 1) ? e[l - 1] : phi;
    for (size_t i = 0; i < n; ++i) dbuf[l - 1][i] += skip[i];
    dl = dbuf[l - 1];
  }
  /* ---- output ---- */
  for (size_t q = 0; q < P; ++q)
    for (int o = 0; o < 3; ++o) {
      double acc = Ob[o];
      for (int i = 0; i < c[0]; ++i) acc += OW[(size_t)o * nO + i] * dbuf[0][q * c[0] + i];
      if (d->r_takes_ld)
        for (int i = 0; i < 3; ++i) acc += OW[(size_t)o * nO + c[0] + i] * direct[q * 3 + i];
      if (dump && dump->logits) dump->logits[q * 3 + o] = acc;
      out[q * 3 + o] = 1.0 / (1.0 + exp(-acc));
    }

  if (dump) {
    if (dump->x) memcpy(dump->x, x, sizeof(double) * P * nx);
    for (int l = 0; l < L; ++l)
      if (dump->e[l]) memcpy(dump->e[l], e[l], sizeof(double) * (size_t)Hl[l] * Wl[l] * c[l]);
    if (dump->tau) memcpy(dump->tau, tau, sizeof(double) * P * (h + 1));
    if (dump->phi) memcpy(dump->phi, phi, sizeof(double) * P * c[0]);
    for (int l = 1; l < L; ++l)
      if (dump->y[l]) memcpy(dump->y[l], ybuf[l], sizeof(double) * (size_t)Hl[l] * Wl[l] * c[l - 1]);
    for (int l = 0; l < L - 1; ++l)
      if (dump->d[l]) memcpy(dump->d[l], dbuf[l], sizeof(double) * (size_t)Hl[l] * Wl[l] * c[l]);
  }
  free(x); free(tau); free(phi);
  for (int l = 0; l < L; ++l) free(e[l]);
  for (int l = 0; l < 4; ++l) { free(dbuf[l]); free(ybuf[l]); }
  return 0;
}

/* ---- N3: the x2 super-sampling network S (§3.4 P:384-389 "a
 * multi-layer CNN is used as a super-sampling network that super-samples the result at x2
 * the original resolution", P:387-389 high-resolution G-buffers are cheap to rasterise;
 * the architecture is unspecified, so SPEC.md's form: the nearest-upsampled
 * image concatenated with the hi-res G-buffer channels -> a shallow CNN -> a residual added
 * to the upsampled image).  DESIGN.md reading N3:
 *   u   = up_nearest(img)                    u[Y][X] = img[Y/2][X/2]          (2H x 2W x 3)
 *   x   = [G'_hi, u]                         G' normalised as in step 1 (R9)  (15 ch)
 *   s1  = ReLU(conv3x3_s1(x;  S1))           15 -> s
 *   s2  = ReLU(conv3x3_s1(s1; S2))           s  -> s
 *   r   = S3.W s2 + S3.b                     1x1, s -> 3
 *   out = clamp(u + r, 0, 1)                 the display image in GlassNet's [0,1] range
 * Weights (fp64, blob order): S1.W[s][3][3][15] S1.b[s] S2.W[s][3][3][s] S2.b[s] S3.W[3][s] S3.b[3].
 * img [H][W][3], gbuf_hi [2H][2W][12], out [2H][2W][3].  Returns 0 on success. */
size_t og_ss_weight_count(int s) { return (size_t)s * 9 * 15 + s + (size_t)s * 9 * s + s + (size_t)3 * s + 3; }

int og_supersample(int H, int W, int s, int input_norm, const double* wts, const double* img,
                   const double* gbuf_hi, double* out) {
  if (H < 1 || W < 1 || s < 1) return 1;
  const int H2 = 2 * H, W2 = 2 * W;
  const size_t P2 = (size_t)H2 * W2;
  const double* p = wts;
  const double* S1W = p; p += (size_t)s * 9 * 15; const double* S1b = p; p += s;
  const double* S2W = p; p += (size_t)s * 9 * s;  const double* S2b = p; p += s;
  const double* S3W = p; p += (size_t)3 * s;      const double* S3b = p;
  double* x = (double*)malloc(sizeof(double) * P2 * 15);
  double* u = (double*)malloc(sizeof(double) * P2 * 3);
  double* s1 = (double*)malloc(sizeof(double) * P2 * s);
  double* s2 = (double*)malloc(sizeof(double) * P2 * s);
  for (int Y = 0; Y < H2; ++Y)
    for (int X = 0; X < W2; ++X) {
      const size_t q = (size_t)Y * W2 + X;
      const size_t qc = (size_t)(Y / 2) * W + (X / 2);       /* nearest: the covering coarse pixel */
      for (int i = 0; i < 3; ++i) u[q * 3 + i] = img[qc * 3 + i];
      for (int i = 0; i < 12; ++i) x[q * 15 + i] = gbuf_hi[q * 12 + i];
      if (input_norm) {
        for (int i = 0; i < 3; ++i) x[q * 15 + i] = x[q * 15 + i] * 0x1p-3;
        x[q * 15 + 11] = x[q * 15 + 11] * 0x1p-7;
      }
      for (int i = 0; i < 3; ++i) x[q * 15 + 12 + i] = u[q * 3 + i];
    }
  og_conv3x3(x, H2, W2, 15, S1W, S1b, s, 1, 1, s1);
  og_conv3x3(s1, H2, W2, s, S2W, S2b, s, 1, 1, s2);
  for (size_t q = 0; q < P2; ++q)
    for (int o = 0; o < 3; ++o) {
      double r = S3b[o];
      for (int i = 0; i < s; ++i) r += S3W[(size_t)o * s + i] * s2[q * s + i];
      double v = u[q * 3 + o] + r;
      out[q * 3 + o] = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    }
  free(x); free(u); free(s1); free(s2);
  return 0;
}

/* One frame. gbuf [H][W][12], direct [H][W][3], tbuf [H][W][K][11], tcount [H][W].
 * out [H][W][3] in [0,1].  Returns 0 on success. */
int og_forward(const og_dims* d, const double* wts, const double* gbuf, const double* direct,
               const double* tbuf, const uint8_t* tcount, double* out, const og_dump* dump) {
  return og_forward_impl(d, wts, gbuf, direct, tbuf, tcount, 0, out, dump);
}

/* N4: one frame from t object buffers (obj[i] [H][W][11], cover[i] [H][W]); d->objects = 1. */
int og_forward_objects(const og_dims* d, const double* wts, const double* gbuf, const double* direct, int t,
                       const double* const* obj, const uint8_t* const* cover, double* out, const og_dump* dump) {
  og_objects ob = {t, obj, cover};
  return og_forward_impl(d, wts, gbuf, direct, 0, 0, &ob, out, dump);
}
