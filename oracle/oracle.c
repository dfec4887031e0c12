/*
 * oracle.c -- plain, slow, fp64 CPU oracle of the padded GPT layer stack and of
 * its DRCE / tensor-parallel re-arrangements.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  It
 * shares no code, header, table or helper with the CUDA path
 * (paper_2209_02341_b200/csrc); the only common module is synth/ (input
 * generation, none of the method's arithmetic).
 *
 * Citations: PAPER.md = /root/reference/PAPER.md (LaTeX source of arXiv
 * 2209.02341), SPEC.md = the CPU-program specification written from it.
 * Readings of points the paper leaves open are SURVEY.md 8(c) C1-C20 and are
 * listed in DESIGN.md ("Readings").
 *
 * Conventions
 *   - every scalar is double; summation over the contraction index runs in
 *     ascending order ("fixed left-to-right over k");
 *   - matrices are [in, out] row-major: y = x W + b;
 *   - per-layer weight pointer order (16): wq wk wv wo bq bk bv bo w1 b1 w2 b2
 *     ln1_g ln1_b ln2_g ln2_b  (= energon_layer_weights order);
 *   - activations in the padded layout are [B, S, H]; head i owns columns
 *     [i*d, (i+1)*d) of Q, K, V.
 *
 * Parity pins for every function are in tests/test_oracle.py; none is
 * "parity unpinned" except where DESIGN.md says so.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int32_t L;       /* layers */
  int32_t H;       /* hidden */
  int32_t h;       /* heads */
  int32_t F;       /* ffn (4H) */
  int32_t causal;  /* PAPER.md:137 "casual mask"; 1 for GPT */
  double eps;      /* LayerNorm eps */
} oracle_cfg;

enum { W_Q, W_K, W_V, W_O, B_Q, B_K, B_V, B_O, W_1, B_1, W_2, B_2, LN1_G, LN1_B, LN2_G, LN2_B, W_COUNT };

/* ------------------------------------------------------------------ primitives */

/* SPEC.md:44-53 matmul: C[m,n] = sum_k A[m,k] W[k,n], k ascending. */
void oracle_matmul(const double* A, const double* W, int64_t M, int64_t K, int64_t N, double* C) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < M; ++i) {
    double* c = C + i * N;
    for (int64_t j = 0; j < N; ++j) c[j] = 0.0;
    for (int64_t k = 0; k < K; ++k) {
      const double a = A[i * K + k];
      const double* w = W + k * N;
      for (int64_t j = 0; j < N; ++j) c[j] += a * w[j];
    }
  }
}

/* y = x W + b  (b may be NULL) */
static void linear(const double* X, const double* W, const double* b, int64_t M, int64_t K, int64_t N,
                   double* Y) {
  oracle_matmul(X, W, M, K, N, Y);
  if (b) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < M; ++i)
      for (int64_t j = 0; j < N; ++j) Y[i * N + j] += b[j];
  }
}

/* SPEC.md:55-63 layer_norm; biased variance (divide by H), eps inside sqrt. */
void oracle_layernorm(const double* x, int64_t rows, int64_t H, const double* g, const double* b, double eps,
                      double* y) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r) {
    const double* xr = x + r * H;
    double mean = 0.0;
    for (int64_t j = 0; j < H; ++j) mean += xr[j];
    mean /= (double)H;
    double var = 0.0;
    for (int64_t j = 0; j < H; ++j) var += (xr[j] - mean) * (xr[j] - mean);
    var /= (double)H;
    const double inv = 1.0 / sqrt(var + eps);
    for (int64_t j = 0; j < H; ++j) y[r * H + j] = (xr[j] - mean) * inv * g[j] + b[j];
  }
}

/* SPEC.md:85-93 GELU, tanh approximation with the fixed constants. */
double oracle_gelu(double x) {
  return 0.5 * x * (1.0 + tanh(0.7978845608 * (x + 0.044715 * x * x * x)));
}

/* Is key t visible from query s of a sequence of valid length len?
 * t < len and (not causal or t <= s). */
static int allowed(int s, int t, int len, int causal) { return t < len && (!causal || t <= s); }

/*
 * SPEC.md:65-83 masked softmax + multi-head attention core.
 * Q, K, V, C: [B, S, H] padded; head i = columns [i*d,(i+1)*d); scale 1/sqrt(d)
 * (SURVEY.md C6).  Masked probabilities are exactly 0 (C7).  Rows of queries
 * s >= len are computed too (the padded oracle); they are never compared.
 */
void oracle_attention(const double* Q, const double* K, const double* V, int B, int S, int H, int h,
                      const int* lens, int causal, double* C) {
  const int d = H / h;
  const double scale = 1.0 / sqrt((double)d);
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int b = 0; b < B; ++b) {
    for (int i = 0; i < h; ++i) {
      double* p = (double*)malloc(sizeof(double) * (size_t)S);
      for (int s = 0; s < S; ++s) {
        const double* q = Q + ((int64_t)b * S + s) * H + (int64_t)i * d;
        double m = -INFINITY;
        for (int t = 0; t < S; ++t) {
          if (!allowed(s, t, lens[b], causal)) { p[t] = 0.0; continue; }
          const double* k = K + ((int64_t)b * S + t) * H + (int64_t)i * d;
          double dot = 0.0;
          for (int j = 0; j < d; ++j) dot += q[j] * k[j];
          p[t] = dot * scale;
          if (p[t] > m) m = p[t];
        }
        double den = 0.0;
        for (int t = 0; t < S; ++t) {
          if (!allowed(s, t, lens[b], causal)) continue;
          p[t] = exp(p[t] - m);
          den += p[t];
        }
        double* c = C + ((int64_t)b * S + s) * H + (int64_t)i * d;
        for (int j = 0; j < d; ++j) c[j] = 0.0;
        if (den == 0.0) continue; /* query with no visible key: only pad queries with causal=0 never; len>=1 */
        for (int t = 0; t < S; ++t) {
          if (!allowed(s, t, lens[b], causal)) continue;
          const double w = p[t] / den;
          const double* v = V + ((int64_t)b * S + t) * H + (int64_t)i * d;
          for (int j = 0; j < d; ++j) c[j] += w * v[j];
        }
      }
      free(p);
    }
  }
}

/* ------------------------------------------------------------------ DRCE index maps */

/*
 * PAPER.md:368-373 (sec 4.3): workers derive the padding layout from seq_lens;
 * SPEC.md:446-466 PackedActivations.  Closed form:
 *   offsets[b] = sum_{i<b} lens[i];  pack_idx[offsets[b]+s] = b*S+s;  pos[...] = s;
 *   unpack_idx[b*S+s] = offsets[b]+s if s < lens[b] else -1.
 * Returns T = offsets[B].
 */
int64_t oracle_index_maps(const int* lens, int B, int S, int* offsets, int* pack_idx, int* pos, int* unpack_idx) {
  int64_t acc = 0;
  for (int b = 0; b < B; ++b) {
    offsets[b] = (int)acc;
    for (int s = 0; s < S; ++s) {
      if (s < lens[b]) {
        pack_idx[acc + s] = b * S + s;
        pos[acc + s] = s;
        unpack_idx[b * S + s] = (int)(acc + s);
      } else {
        unpack_idx[b * S + s] = -1;
      }
    }
    acc += lens[b];
  }
  offsets[B] = (int)acc;
  return acc;
}

/* ------------------------------------------------------------------ the padded layer */

/*
 * One pre-LN GPT layer on the padded batch, in place on X [B,S,H]
 * (PAPER.md:143-149 fig:transformer):
 *   A = LN1(X); Q,K,V = A Wq+bq, A Wk+bk, A Wv+bv; C = attn(Q,K,V)
 *   X = X + C Wo + bo
 *   X = X + gelu(LN2(X) W1 + b1) W2 + b2
 */
void oracle_layer_padded(const oracle_cfg* cfg, const double* const* w, double* X, const int* lens, int B, int S) {
  const int64_t M = (int64_t)B * S, H = cfg->H, F = cfg->F;
  double* A = (double*)malloc(sizeof(double) * M * H);
  double* Q = (double*)malloc(sizeof(double) * M * H);
  double* K = (double*)malloc(sizeof(double) * M * H);
  double* V = (double*)malloc(sizeof(double) * M * H);
  double* C = (double*)malloc(sizeof(double) * M * H);
  double* G = (double*)malloc(sizeof(double) * M * F);
  oracle_layernorm(X, M, H, w[LN1_G], w[LN1_B], cfg->eps, A);
  linear(A, w[W_Q], w[B_Q], M, H, H, Q);
  linear(A, w[W_K], w[B_K], M, H, H, K);
  linear(A, w[W_V], w[B_V], M, H, H, V);
  oracle_attention(Q, K, V, B, S, (int)H, cfg->h, lens, cfg->causal, C);
  linear(C, w[W_O], w[B_O], M, H, H, A); /* A <- attention branch */
  for (int64_t i = 0; i < M * H; ++i) X[i] += A[i];
  oracle_layernorm(X, M, H, w[LN2_G], w[LN2_B], cfg->eps, A);
  linear(A, w[W_1], w[B_1], M, H, F, G);
  for (int64_t i = 0; i < M * F; ++i) G[i] = oracle_gelu(G[i]);
  linear(G, w[W_2], w[B_2], M, F, H, A);
  for (int64_t i = 0; i < M * H; ++i) X[i] += A[i];
  free(A); free(Q); free(K); free(V); free(C); free(G);
}

/* X[b,s] = E[tok[b,s]] + P[s] for every s < S (pad tokens use id 0, C12). */
void oracle_embed(const oracle_cfg* cfg, const double* tok_emb, const double* pos_emb, const int* tok, int B,
                  int S, double* X) {
  const int64_t H = cfg->H;
  for (int64_t r = 0; r < (int64_t)B * S; ++r) {
    const int s = (int)(r % S);
    for (int64_t j = 0; j < H; ++j) X[r * H + j] = tok_emb[(int64_t)tok[r] * H + j] + pos_emb[(int64_t)s * H + j];
  }
}

/* Layers [l0, l1) on the padded residual stream X [B,S,H] (teacher-forced per-layer parity). */
void oracle_layers_padded(const oracle_cfg* cfg, const double* const* layer_w, int l0, int l1, double* X,
                          const int* lens, int B, int S) {
  for (int l = l0; l < l1; ++l) oracle_layer_padded(cfg, layer_w + (int64_t)l * W_COUNT, X, lens, B, S);
}

/*
 * SPEC.md:147-155 serial_forward: embedding -> L layers -> final LN (SURVEY.md
 * 8(c) "Plain definition").  Y [B,S,H]; only s < lens[b] is meaningful.
 */
void oracle_forward_padded(const oracle_cfg* cfg, const double* const* layer_w, const double* tok_emb,
                           const double* pos_emb, const double* lnf_g, const double* lnf_b, const int* tok,
                           const int* lens, int B, int S, int final_ln, double* Y) {
  const int64_t M = (int64_t)B * S, H = cfg->H;
  double* X = (double*)malloc(sizeof(double) * M * H);
  oracle_embed(cfg, tok_emb, pos_emb, tok, B, S, X);
  oracle_layers_padded(cfg, layer_w, 0, cfg->L, X, lens, B, S);
  if (final_ln) oracle_layernorm(X, M, H, lnf_g, lnf_b, cfg->eps, Y);
  else memcpy(Y, X, sizeof(double) * M * H);
  free(X);
}

/* ------------------------------------------------------------------ DRCE companion */

/*
 * PAPER.md:358-373 (sec 4.3, fig:drce) as read in SURVEY.md C1/C2: remove
 * padding once at entry; every LN / linear / residual runs on the T packed rows;
 * Q,K,V are rebuilt into the padded layout for attention ("the multi-head
 * attention module still requires the padding area"), and the attention output
 * is packed again.  The final LN output is unpacked with pad rows = 0
 * (SPEC.md:465).  P10: equals oracle_forward_padded at valid positions.
 */
void oracle_forward_drce(const oracle_cfg* cfg, const double* const* layer_w, const double* tok_emb,
                         const double* pos_emb, const double* lnf_g, const double* lnf_b, const int* tok,
                         const int* lens, int B, int S, int final_ln, double* Y) {
  const int64_t H = cfg->H, F = cfg->F, BS = (int64_t)B * S;
  int* offsets = (int*)malloc(sizeof(int) * (B + 1));
  int* pack_idx = (int*)malloc(sizeof(int) * BS);
  int* pos = (int*)malloc(sizeof(int) * BS);
  int* unpack_idx = (int*)malloc(sizeof(int) * BS);
  const int64_t T = oracle_index_maps(lens, B, S, offsets, pack_idx, pos, unpack_idx);
  double* X = (double*)malloc(sizeof(double) * T * H);
  double* A = (double*)malloc(sizeof(double) * T * H);
  double* Qp = (double*)malloc(sizeof(double) * T * H);
  double* Kp = (double*)malloc(sizeof(double) * T * H);
  double* Vp = (double*)malloc(sizeof(double) * T * H);
  double* G = (double*)malloc(sizeof(double) * T * F);
  double* Qd = (double*)calloc((size_t)(BS * H), sizeof(double));
  double* Kd = (double*)calloc((size_t)(BS * H), sizeof(double));
  double* Vd = (double*)calloc((size_t)(BS * H), sizeof(double));
  double* Cd = (double*)calloc((size_t)(BS * H), sizeof(double));
  /* remove padding at entry: gather only the valid rows (C2, C12) */
  for (int64_t t = 0; t < T; ++t) {
    const int r = pack_idx[t];
    for (int64_t j = 0; j < H; ++j) X[t * H + j] = tok_emb[(int64_t)tok[r] * H + j] + pos_emb[(int64_t)pos[t] * H + j];
  }
  for (int l = 0; l < cfg->L; ++l) {
    const double* const* w = layer_w + (int64_t)l * W_COUNT;
    oracle_layernorm(X, T, H, w[LN1_G], w[LN1_B], cfg->eps, A);
    linear(A, w[W_Q], w[B_Q], T, H, H, Qp);
    linear(A, w[W_K], w[B_K], T, H, H, Kp);
    linear(A, w[W_V], w[B_V], T, H, H, Vp);
    /* rebuild padding (paper kernel #1) */
    for (int64_t t = 0; t < T; ++t) {
      const int64_t r = pack_idx[t];
      memcpy(Qd + r * H, Qp + t * H, sizeof(double) * H);
      memcpy(Kd + r * H, Kp + t * H, sizeof(double) * H);
      memcpy(Vd + r * H, Vp + t * H, sizeof(double) * H);
    }
    oracle_attention(Qd, Kd, Vd, B, S, (int)H, cfg->h, lens, cfg->causal, Cd);
    /* remove padding (paper kernel #2) */
    for (int64_t t = 0; t < T; ++t) memcpy(Qp + t * H, Cd + (int64_t)pack_idx[t] * H, sizeof(double) * H);
    linear(Qp, w[W_O], w[B_O], T, H, H, A);
    for (int64_t i = 0; i < T * H; ++i) X[i] += A[i];
    oracle_layernorm(X, T, H, w[LN2_G], w[LN2_B], cfg->eps, A);
    linear(A, w[W_1], w[B_1], T, H, F, G);
    for (int64_t i = 0; i < T * F; ++i) G[i] = oracle_gelu(G[i]);
    linear(G, w[W_2], w[B_2], T, F, H, A);
    for (int64_t i = 0; i < T * H; ++i) X[i] += A[i];
  }
  if (final_ln) oracle_layernorm(X, T, H, lnf_g, lnf_b, cfg->eps, A);
  else memcpy(A, X, sizeof(double) * T * H);
  for (int64_t r = 0; r < BS; ++r) {
    const int t = unpack_idx[r];
    for (int64_t j = 0; j < H; ++j) Y[r * H + j] = (t >= 0) ? A[(int64_t)t * H + j] : 0.0;
  }
  free(offsets); free(pack_idx); free(pos); free(unpack_idx);
  free(X); free(A); free(Qp); free(Kp); free(Vp); free(G); free(Qd); free(Kd); free(Vd); free(Cd);
}

/* ------------------------------------------------------------------ 1-D TP companion */

/* copy columns [c0, c0+n) of a row-major [rows, ld] matrix */
static double* col_slice(const double* W, int64_t rows, int64_t ld, int64_t c0, int64_t n) {
  double* out = (double*)malloc(sizeof(double) * rows * n);
  for (int64_t i = 0; i < rows; ++i) memcpy(out + i * n, W + i * ld + c0, sizeof(double) * n);
  return out;
}

/*
 * PAPER.md:281-293 (sec 4.1.3, fig:transformer1d) 1-D Megatron TP over k ranks,
 * simulated serially on the padded batch:
 *   rank r owns heads [r h/k, (r+1) h/k) -> columns of Wq,Wk,Wv (column-parallel)
 *   and the matching rows of Wo (row-parallel); FFN columns [r F/k, (r+1) F/k)
 *   of W1 and rows of W2 (C10).
 *   Partials are "accumulated by communications": summed in
 *   ascending rank order; row-linear biases are added once after
 *   the sum.  Exactly 2 reductions per layer:
 *   *allreduce_count is incremented for each.
 */
void oracle_forward_tp(const oracle_cfg* cfg, int k, const double* const* layer_w, const double* tok_emb,
                       const double* pos_emb, const double* lnf_g, const double* lnf_b, const int* tok,
                       const int* lens, int B, int S, int final_ln, double* Y, int64_t* allreduce_count) {
  const int64_t M = (int64_t)B * S, H = cfg->H, F = cfg->F, Hk = H / k, Fk = F / k, hk = cfg->h / k;
  double* X = (double*)malloc(sizeof(double) * M * H);
  double* A = (double*)malloc(sizeof(double) * M * H);
  double* Q = (double*)malloc(sizeof(double) * M * Hk);
  double* K = (double*)malloc(sizeof(double) * M * Hk);
  double* V = (double*)malloc(sizeof(double) * M * Hk);
  double* C = (double*)malloc(sizeof(double) * M * Hk);
  double* G = (double*)malloc(sizeof(double) * M * Fk);
  double* part = (double*)malloc(sizeof(double) * k * M * H);
  oracle_embed(cfg, tok_emb, pos_emb, tok, B, S, X);
  for (int l = 0; l < cfg->L; ++l) {
    const double* const* w = layer_w + (int64_t)l * W_COUNT;
    /* attention module: column-parallel QKV, local heads, row-parallel out-proj */
    oracle_layernorm(X, M, H, w[LN1_G], w[LN1_B], cfg->eps, A);
    for (int r = 0; r < k; ++r) {
      double* wq = col_slice(w[W_Q], H, H, r * Hk, Hk);
      double* wk = col_slice(w[W_K], H, H, r * Hk, Hk);
      double* wv = col_slice(w[W_V], H, H, r * Hk, Hk);
      linear(A, wq, w[B_Q] + r * Hk, M, H, Hk, Q);
      linear(A, wk, w[B_K] + r * Hk, M, H, Hk, K);
      linear(A, wv, w[B_V] + r * Hk, M, H, Hk, V);
      oracle_attention(Q, K, V, B, S, (int)Hk, (int)hk, lens, cfg->causal, C);
      /* row shard of Wo: rows [r Hk, (r+1) Hk) = contiguous block */
      linear(C, w[W_O] + r * Hk * H, NULL, M, Hk, H, part + r * M * H);
      free(wq); free(wk); free(wv);
    }
    for (int64_t i = 0; i < M * H; ++i) {
      double s = 0.0;
      for (int r = 0; r < k; ++r) s += part[r * M * H + i];
      X[i] += s + w[B_O][i % H];
    }
    if (allreduce_count) ++*allreduce_count;
    /* MLP module: column-parallel W1, row-parallel W2 */
    oracle_layernorm(X, M, H, w[LN2_G], w[LN2_B], cfg->eps, A);
    for (int r = 0; r < k; ++r) {
      double* w1 = col_slice(w[W_1], H, F, r * Fk, Fk);
      linear(A, w1, w[B_1] + r * Fk, M, H, Fk, G);
      for (int64_t i = 0; i < M * Fk; ++i) G[i] = oracle_gelu(G[i]);
      linear(G, w[W_2] + r * Fk * H, NULL, M, Fk, H, part + r * M * H);
      free(w1);
    }
    for (int64_t i = 0; i < M * H; ++i) {
      double s = 0.0;
      for (int r = 0; r < k; ++r) s += part[r * M * H + i];
      X[i] += s + w[B_2][i % H];
    }
    if (allreduce_count) ++*allreduce_count;
  }
  if (final_ln) oracle_layernorm(X, M, H, lnf_g, lnf_b, cfg->eps, Y);
  else memcpy(Y, X, sizeof(double) * M * H);
  free(X); free(A); free(Q); free(K); free(V); free(C); free(G); free(part);
}

/* Number of threads OpenMP will use (reported as cpu_baseline.cores). */
int oracle_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}
