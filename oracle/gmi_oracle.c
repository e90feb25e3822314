/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle.  Never linked into, called by,
 * or shipped with the product path (paper_2012_13257_b200/).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load it, and only as the checker.
 *
 * A plain-C restatement of the reference's hot path
 * (/root/reference/proj, C++20, f64 throughout), following it statement by
 * statement so that for C in {1,3} it reproduces the reference bit for bit
 * (pinned against oracle/_ref — the reference compiled from its own
 * sources — and against tests/golden/, see tests/test_oracle.py).
 * Compiled with -ffp-contract=off so no FMA contraction changes rounding.
 *
 * Generalisation beyond the reference: any channel count C >= 1 (the
 * reference rejects C not in {1,3}, core.cpp:60-64).  Channels are
 * independent in every formula, so per-channel results equal the
 * reference's per-channel-group runs.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- core.cpp:49-53 gaussian_weight ----------------------------------- */
double orc_gaussian_weight(double qx, double qy, double mx, double my,
                           double sigma) {
    const double dx = qx - mx;
    const double dy = qy - my;
    return exp(-(dx * dx + dy * dy) / (2.0 * sigma * sigma));
}

/* ---- core.hpp:35-50 ErrorCode values (0-based), returned +1 ----------- */
enum {
    ORC_NonFiniteValue = 0,
    ORC_ColorOutOfRange = 1,
    ORC_EmptyPointSet = 2,
    ORC_ShapeMismatch = 3,
    ORC_InvalidCellSize = 4,
    ORC_ConfigInvalid = 5,
    ORC_CacheMismatch = 6,
    ORC_InvalidDimensions = 7,
};

/* core.cpp:55-96 validate_point_set (C range relaxed to C >= 1).  Returns
 * 0 when valid, else 1 + ErrorCode; *index = offending point or -1. */
int orc_validate(const double* pos, const double* col, int n, int channels,
                 long* index) {
    *index = -1;
    if (n <= 0) return 1 + ORC_EmptyPointSet;
    if (channels < 1) return 1 + ORC_ShapeMismatch;
    for (int i = 0; i < n; ++i) {
        if (!isfinite(pos[2 * i]) || !isfinite(pos[2 * i + 1])) {
            *index = i;
            return 1 + ORC_NonFiniteValue;
        }
        for (int ch = 0; ch < channels; ++ch) {
            const double c = col[(size_t)i * channels + ch];
            if (!isfinite(c)) {
                *index = i;
                return 1 + ORC_NonFiniteValue;
            }
            if (c < 0.0 || c > 1.0) {
                *index = i;
                return 1 + ORC_ColorOutOfRange;
            }
        }
    }
    return 0;
}

/* ---- bin_grid.cpp:14-36 ------------------------------------------------ */
/* (int)floor(v) as the reference's x86-64 build executes it: cvttsd2si
 * yields INT_MIN for NaN / out-of-range values. */
static int x86_double_to_int(double v) {
    if (!(v >= -2147483648.0 && v < 2147483648.0)) return INT32_MIN;
    return (int)v;
}

static int clamp_int(int v, int lo, int hi) {
    return v < lo ? lo : (v > hi ? hi : v);
}

/* axis_cells with a configurable cap (reference: 2048, bin_grid.cpp:14) */
int orc_axis_cells(double span, double cell, int cap) {
    const double ideal = ceil(span / cell) + 2.0;
    if (!(ideal < (double)cap)) return cap;
    const int v = x86_double_to_int(ideal);
    return v > 1 ? v : 1;
}

typedef struct {
    double cell;
    double ox, oy;
    int n_cols, n_rows;
} orc_grid_geom;

static int cell_of(double v, double o, double cell, int n) {
    return clamp_int(x86_double_to_int(floor((v - o) / cell)), 0, n - 1);
}

/* build_bin_grid geometry (bin_grid.cpp:45-60) */
static orc_grid_geom grid_geometry(const double* pos, int n, double cell,
                                   int cap) {
    double min_x = INFINITY, min_y = INFINITY;
    double max_x = -INFINITY, max_y = -INFINITY;
    for (int i = 0; i < n; ++i) {
        /* std::min(a,b) = (b < a) ? b : a ; std::max(a,b) = (a < b) ? b : a */
        if (pos[2 * i] < min_x) min_x = pos[2 * i];
        if (pos[2 * i + 1] < min_y) min_y = pos[2 * i + 1];
        if (max_x < pos[2 * i]) max_x = pos[2 * i];
        if (max_y < pos[2 * i + 1]) max_y = pos[2 * i + 1];
    }
    orc_grid_geom g;
    g.cell = cell;
    g.ox = min_x - cell;
    g.oy = min_y - cell;
    g.n_cols = orc_axis_cells(max_x - min_x, cell, cap);
    g.n_rows = orc_axis_cells(max_y - min_y, cell, cap);
    return g;
}

/* build_bin_grid dims: origin[2], n_cols, n_rows.  cap=2048 reproduces the
 * reference exactly. */
int orc_bin_grid_dims(const double* pos, int n, double cell, int cap,
                      double* origin, int* n_cols, int* n_rows) {
    if (!isfinite(cell) || cell <= 0.0) return 1 + ORC_InvalidCellSize;
    if (n <= 0) return 1 + ORC_EmptyPointSet;
    const orc_grid_geom g = grid_geometry(pos, n, cell, cap);
    origin[0] = g.ox;
    origin[1] = g.oy;
    *n_cols = g.n_cols;
    *n_rows = g.n_rows;
    return 0;
}

/* build_bin_grid CSR (bin_grid.cpp:62-81): bin_start[n_bins+1],
 * point_index[n]; stable ascending fill. */
int orc_bin_grid_fill(const double* pos, int n, double cell, int cap,
                      int* bin_start, int* point_index) {
    if (!isfinite(cell) || cell <= 0.0) return 1 + ORC_InvalidCellSize;
    const orc_grid_geom g = grid_geometry(pos, n, cell, cap);
    const int n_bins = g.n_cols * g.n_rows;
    int* cell_of_pt = (int*)malloc(sizeof(int) * (size_t)n);
    int* cursor = (int*)calloc((size_t)n_bins + 1, sizeof(int));
    memset(bin_start, 0, sizeof(int) * ((size_t)n_bins + 1));
    for (int i = 0; i < n; ++i) {
        const int b = cell_of(pos[2 * i + 1], g.oy, cell, g.n_rows) * g.n_cols +
                      cell_of(pos[2 * i], g.ox, cell, g.n_cols);
        cell_of_pt[i] = b;
        bin_start[b + 1]++;
    }
    for (int b = 0; b < n_bins; ++b) bin_start[b + 1] += bin_start[b];
    memcpy(cursor, bin_start, sizeof(int) * (size_t)n_bins);
    for (int i = 0; i < n; ++i) point_index[cursor[cell_of_pt[i]]++] = i;
    free(cell_of_pt);
    free(cursor);
    return 0;
}

/* ---- internal grid used by the restated forward/backward -------------- */
typedef struct {
    orc_grid_geom g;
    int* bin_start;
    int* point_index;
} orc_grid;

static void grid_build(orc_grid* G, const double* pos, int n, double cell) {
    G->g = grid_geometry(pos, n, cell, 2048);
    const size_t nb = (size_t)G->g.n_cols * G->g.n_rows;
    G->bin_start = (int*)malloc(sizeof(int) * (nb + 1));
    G->point_index = (int*)malloc(sizeof(int) * (size_t)n);
    orc_bin_grid_fill(pos, n, cell, 2048, G->bin_start, G->point_index);
}

static void grid_free(orc_grid* G) {
    free(G->bin_start);
    free(G->point_index);
}

static int cmp_int(const void* a, const void* b) {
    const int x = *(const int*)a, y = *(const int*)b;
    return (x > y) - (x < y);
}

/* query_radius (bin_grid.cpp:84-105): closed ball, ascending indices. */
static int query_radius(const orc_grid* G, const double* pos, double qx,
                        double qy, double radius, int* out) {
    int cnt = 0;
    const double r2 = radius * radius;
    const int cx0 = cell_of(qx - radius, G->g.ox, G->g.cell, G->g.n_cols);
    const int cx1 = cell_of(qx + radius, G->g.ox, G->g.cell, G->g.n_cols);
    const int cy0 = cell_of(qy - radius, G->g.oy, G->g.cell, G->g.n_rows);
    const int cy1 = cell_of(qy + radius, G->g.oy, G->g.cell, G->g.n_rows);
    for (int gy = cy0; gy <= cy1; ++gy) {
        for (int gx = cx0; gx <= cx1; ++gx) {
            const int bin = gy * G->g.n_cols + gx;
            for (int k = G->bin_start[bin]; k < G->bin_start[bin + 1]; ++k) {
                const int i = G->point_index[k];
                const double dx = qx - pos[2 * i];
                const double dy = qy - pos[2 * i + 1];
                if (dx * dx + dy * dy <= r2) out[cnt++] = i;
            }
        }
    }
    qsort(out, (size_t)cnt, sizeof(int), cmp_int);
    return cnt;
}

/* nearest_point (bin_grid.cpp:114-164): Chebyshev ring search, ties to the
 * smallest index, pruned by the (ring-1)*cell lower bound. */
static int nearest_point(const orc_grid* G, const double* pos, double qx,
                         double qy) {
    int best = -1;
    double best_d2 = INFINITY;
    const orc_grid_geom* g = &G->g;
#define ORC_SCAN_CELL(GX, GY)                                                  \
    do {                                                                       \
        const int gx_ = (GX), gy_ = (GY);                                      \
        if (!(gx_ < 0 || gx_ >= g->n_cols || gy_ < 0 || gy_ >= g->n_rows)) {   \
            const int bin_ = gy_ * g->n_cols + gx_;                            \
            for (int k = G->bin_start[bin_]; k < G->bin_start[bin_ + 1]; ++k) { \
                const int i = G->point_index[k];                               \
                const double dx = qx - pos[2 * i], dy = qy - pos[2 * i + 1];  \
                const double d2 = dx * dx + dy * dy;                           \
                if (d2 < best_d2 || (d2 == best_d2 && i < best)) {             \
                    best = i;                                                  \
                    best_d2 = d2;                                              \
                }                                                              \
            }                                                                  \
        }                                                                      \
    } while (0)
    const int qcx = x86_double_to_int(floor((qx - g->ox) / g->cell));
    const int qcy = x86_double_to_int(floor((qy - g->oy) / g->cell));
    const int ax = abs(qcx), bx = abs(qcx - (g->n_cols - 1));
    const int ay = abs(qcy), by = abs(qcy - (g->n_rows - 1));
    const int cap_x = ax > bx ? ax : bx;
    const int cap_y = ay > by ? ay : by;
    const int ring_cap = cap_x > cap_y ? cap_x : cap_y;
    for (int ring = 0; ring <= ring_cap; ++ring) {
        if (best >= 0 && ring >= 1) {
            const double lb = (ring - 1) * g->cell;
            if (lb * lb > best_d2) break;
        }
        if (ring == 0) {
            ORC_SCAN_CELL(qcx, qcy);
            continue;
        }
        for (int gx = qcx - ring; gx <= qcx + ring; ++gx) {
            ORC_SCAN_CELL(gx, qcy - ring);
            ORC_SCAN_CELL(gx, qcy + ring);
        }
        for (int gy = qcy - ring + 1; gy <= qcy + ring - 1; ++gy) {
            ORC_SCAN_CELL(qcx - ring, gy);
            ORC_SCAN_CELL(qcx + ring, gy);
        }
    }
#undef ORC_SCAN_CELL
    return best;
}

/* Exported for the bin-grid tests. */
int orc_query_radius(const double* pos, int n, double cell, double qx,
                     double qy, double radius, int* out) {
    orc_grid G;
    grid_build(&G, pos, n, cell);
    const int cnt = query_radius(&G, pos, qx, qy, radius, out);
    grid_free(&G);
    return cnt;
}

int orc_nearest_point(const double* pos, int n, double cell, double qx,
                      double qy) {
    orc_grid G;
    grid_build(&G, pos, n, cell);
    const int r = nearest_point(&G, pos, qx, qy);
    grid_free(&G);
    return r;
}

static int check_cfg(double sigma, double cutoff, int width, int height) {
    if (!isfinite(sigma) || sigma <= 0.0) return 1 + ORC_ConfigInvalid;
    if (!isfinite(cutoff) || cutoff <= 0.0) return 1 + ORC_ConfigInvalid;
    if (width < 1 || height < 1) return 1 + ORC_InvalidDimensions;
    return 0;
}

/* ---- engine.cpp:44-176 forward ----------------------------------------
 * Outputs (any may be NULL except image):
 *   image[H*W*C], normalizer[H*W], fallback_flag[H*W], nearest_index[H*W],
 *   counts[H*W] = contributions per pixel (pixel_start deltas).
 * fallback: 0 = NearestPoint, 1 = Zero.  Returns 0 or 1 + ErrorCode. */
int orc_forward(const double* pos, const double* col, int n, int channels,
                int width, int height, double sigma, double cutoff,
                int fallback, double* image, double* normalizer,
                uint8_t* fallback_flag, int* nearest_index, int64_t* counts) {
    long bad;
    int err = orc_validate(pos, col, n, channels, &bad);
    if (err) return err;
    err = check_cfg(sigma, cutoff, width, height);
    if (err) return err;
    orc_grid G;
    grid_build(&G, pos, n, cutoff); /* engine.cpp:115 */
    int* nb = (int*)malloc(sizeof(int) * (size_t)n);
    double* num = (double*)malloc(sizeof(double) * (size_t)channels);
    for (int r = 0; r < height; ++r) {
        for (int c = 0; c < width; ++c) {
            const double qx = (double)c, qy = (double)r;
            const int64_t pix = (int64_t)r * width + c;
            const int cnt = query_radius(&G, pos, qx, qy, cutoff, nb);
            double wsum = 0.0;
            for (int ch = 0; ch < channels; ++ch) num[ch] = 0.0;
            for (int k = 0; k < cnt; ++k) {
                const int i = nb[k];
                const double w = orc_gaussian_weight(qx, qy, pos[2 * i],
                                                     pos[2 * i + 1], sigma);
                wsum += w;
                for (int ch = 0; ch < channels; ++ch)
                    num[ch] += col[(size_t)i * channels + ch] * w;
            }
            double* out = image + (size_t)pix * channels;
            if (wsum <= 0.0) {
                if (counts) counts[pix] = 0;
                if (fallback_flag) fallback_flag[pix] = 1;
                if (normalizer) normalizer[pix] = 0.0;
                if (fallback == 0) {
                    const int j = nearest_point(&G, pos, qx, qy);
                    if (nearest_index) nearest_index[pix] = j;
                    for (int ch = 0; ch < channels; ++ch)
                        out[ch] = col[(size_t)j * channels + ch];
                } else {
                    if (nearest_index) nearest_index[pix] = -1;
                    for (int ch = 0; ch < channels; ++ch) out[ch] = 0.0;
                }
            } else {
                if (counts) counts[pix] = cnt;
                if (fallback_flag) fallback_flag[pix] = 0;
                if (nearest_index) nearest_index[pix] = -1;
                if (normalizer) normalizer[pix] = wsum;
                for (int ch = 0; ch < channels; ++ch) out[ch] = num[ch] / wsum;
            }
        }
    }
    free(num);
    free(nb);
    grid_free(&G);
    return 0;
}

/* ---- engine.cpp:12-23 row_ranges -------------------------------------- */
static void row_range(int height, int workers, int w, int* begin, int* end) {
    const int chunk = (height + workers - 1) / workers;
    int b = w * chunk;
    if (b > height) b = height;
    int e = b + chunk;
    if (e > height) e = height;
    *begin = b;
    *end = e;
}

/* ---- engine.cpp:190-309 backward ---------------------------------------
 * Recomputes the forward's neighbour lists (query_radius is deterministic,
 * so the (i, w) sequence equals the reference's cached CSR) and reproduces
 * the min(H,16) row-slot partials summed in slot order (engine.cpp:252-307).
 * image/normalizer/fallback_flag/nearest_index: the forward outputs. */
int orc_backward(const double* pos, const double* col, int n, int channels,
                 int width, int height, double sigma, double cutoff,
                 int fallback, const double* image, const double* normalizer,
                 const uint8_t* fallback_flag, const int* nearest_index,
                 const double* upstream, double* d_colors,
                 double* d_positions) {
    long bad;
    int err = orc_validate(pos, col, n, channels, &bad);
    if (err) return err;
    err = check_cfg(sigma, cutoff, width, height);
    if (err) return err;
    orc_grid G;
    grid_build(&G, pos, n, cutoff);
    const int num_slots = height < 16 ? height : 16;
    const double inv_sigma2 = 1.0 / (sigma * sigma);
    const size_t nc = (size_t)n * channels;
    double* pc = (double*)malloc(sizeof(double) * nc);
    double* pp = (double*)malloc(sizeof(double) * 2 * (size_t)n);
    int* nb = (int*)malloc(sizeof(int) * (size_t)n);
    memset(d_colors, 0, sizeof(double) * nc);
    memset(d_positions, 0, sizeof(double) * 2 * (size_t)n);
    for (int s = 0; s < num_slots; ++s) {
        int r0, r1;
        row_range(height, num_slots, s, &r0, &r1);
        memset(pc, 0, sizeof(double) * nc);
        memset(pp, 0, sizeof(double) * 2 * (size_t)n);
        for (int r = r0; r < r1; ++r) {
            for (int c = 0; c < width; ++c) {
                const int64_t pix = (int64_t)r * width + c;
                const double* up = upstream + (size_t)pix * channels;
                if (fallback_flag[pix]) {
                    if (fallback == 0) {
                        const int j = nearest_index[pix];
                        for (int ch = 0; ch < channels; ++ch)
                            pc[(size_t)j * channels + ch] += up[ch];
                    }
                    continue;
                }
                const double qx = (double)c, qy = (double)r;
                const double inv_w = 1.0 / normalizer[pix];
                const int cnt = query_radius(&G, pos, qx, qy, cutoff, nb);
                for (int k = 0; k < cnt; ++k) {
                    const int i = nb[k];
                    const double w = orc_gaussian_weight(qx, qy, pos[2 * i],
                                                         pos[2 * i + 1], sigma);
                    const double ratio = w * inv_w;
                    double dot = 0.0;
                    for (int ch = 0; ch < channels; ++ch) {
                        pc[(size_t)i * channels + ch] += up[ch] * ratio;
                        dot += up[ch] * (col[(size_t)i * channels + ch] -
                                         image[(size_t)pix * channels + ch]);
                    }
                    const double coef = ratio * dot * inv_sigma2;
                    pp[2 * i] += coef * (qx - pos[2 * i]);
                    pp[2 * i + 1] += coef * (qy - pos[2 * i + 1]);
                }
            }
        }
        for (size_t k = 0; k < nc; ++k) d_colors[k] += pc[k];
        for (int i = 0; i < n; ++i) {
            d_positions[2 * i] += pp[2 * i];
            d_positions[2 * i + 1] += pp[2 * i + 1];
        }
    }
    free(nb);
    free(pp);
    free(pc);
    grid_free(&G);
    return 0;
}

/* ---- rng.hpp:12-59 xoshiro256++ seeded by splitmix64 ------------------ */
typedef struct {
    uint64_t s[4];
} orc_rng;

static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

void orc_rng_seed(orc_rng* r, uint64_t seed) {
    uint64_t x = seed;
    for (int k = 0; k < 4; ++k) {
        x += 0x9E3779B97F4A7C15ULL;
        uint64_t z = x;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        r->s[k] = z ^ (z >> 31);
    }
}

uint64_t orc_rng_next(orc_rng* r) {
    uint64_t* s = r->s;
    const uint64_t result = rotl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
}

static double rng_double(orc_rng* r) {
    return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53;
}

static double rng_uniform(orc_rng* r, double lo, double hi) {
    return lo + (hi - lo) * rng_double(r);
}

void orc_rng_u64(uint64_t seed, int k, uint64_t* out) {
    orc_rng r;
    orc_rng_seed(&r, seed);
    for (int i = 0; i < k; ++i) out[i] = orc_rng_next(&r);
}

/* Synthetic batch inputs per SURVEY.md §8(d): master = Rng(seed), per image
 * Rng(master.next_u64()); x = (float)U(-0.5, W-0.5), y = (float)U(-0.5,
 * H-0.5) (the random_subsample rectangle, imaging.cpp:362-363); colours
 * (float)U[0,1); the first floor(cluster_frac*N) points uniform in a
 * cluster_px square at ((float)U(0,W-cluster_px), (float)U(0,H-cluster_px)).
 * Each image draws two master outputs: its point seed and its upstream
 * seed; upstream is (float)U(-1,1) (validate.cpp:37-44) when != NULL. */
void orc_synth_batch(uint64_t seed, int batch, int n, int channels, int width,
                     int height, double cluster_frac, int cluster_px,
                     float* pos, float* col, float* upstream) {
    orc_rng master;
    orc_rng_seed(&master, seed);
    for (int b = 0; b < batch; ++b) {
        orc_rng r;
        const uint64_t seed_points = orc_rng_next(&master);
        const uint64_t seed_upstream = orc_rng_next(&master);
        orc_rng_seed(&r, seed_points);
        float* p = pos + (size_t)b * n * 2;
        float* c = col + (size_t)b * n * channels;
        const int n_cluster = (int)floor(cluster_frac * n);
        double cx = 0.0, cy = 0.0;
        if (n_cluster > 0) {
            cx = (float)rng_uniform(&r, 0.0, (double)(width - cluster_px));
            cy = (float)rng_uniform(&r, 0.0, (double)(height - cluster_px));
        }
        for (int i = 0; i < n; ++i) {
            if (i < n_cluster) {
                p[2 * i] = (float)(cx + rng_uniform(&r, 0.0, cluster_px));
                p[2 * i + 1] = (float)(cy + rng_uniform(&r, 0.0, cluster_px));
            } else {
                p[2 * i] = (float)rng_uniform(&r, -0.5, width - 0.5);
                p[2 * i + 1] = (float)rng_uniform(&r, -0.5, height - 0.5);
            }
            for (int ch = 0; ch < channels; ++ch)
                c[(size_t)i * channels + ch] = (float)rng_double(&r);
        }
        if (upstream != NULL) {
            orc_rng u;
            orc_rng_seed(&u, seed_upstream);
            float* up = upstream + (size_t)b * height * width * channels;
            const size_t m = (size_t)height * width * channels;
            for (size_t k = 0; k < m; ++k) up[k] = (float)rng_uniform(&u, -1.0, 1.0);
        }
    }
}
