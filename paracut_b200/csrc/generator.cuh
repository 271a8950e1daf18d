// generator.cuh -- the BASELINE synthetic instances built in HBM
// (SURVEY.md section 8(f4)); the host reference is paracut_b200/instances.py.
//
// Image I: background 0.3, seeded disks / balls of 0.7 (centres and radii come
// from the host's numpy default_rng(seed) draw, a few hundred numbers), plus
// N(0, 0.15^2) noise from a counter-based stream: node i's value is
// Philox-4x32-10 at counter (i, 0, NOISE_STREAM, 0) under key = seed, a 53-bit
// uniform, and the inverse normal CDF (AS241 / PPND16).  Unaries
// w = 10 (I - 0.5), pairwise lambda * exp(-(I_i - I_j)^2 / (2 * 0.1^2)) per
// direction (2D-8 diagonals / sqrt 2), integer variant by rint.  log and exp
// are the series of instances.py, every other step integer or IEEE-exact fp64,
// and the translation unit is built with -fmad=false: the arrays equal the
// host reference bit for bit (tests/test_gpu_generator.py).
#pragma once

namespace pcb {
namespace gen {

constexpr uint32_t NOISE_STREAM = 0x6E6F6973u;
constexpr double LN2 = 0.6931471805599453;
constexpr double LN2_HI = 6.93147180369123816490e-01, LN2_LO = 1.90821492927058770002e-10;

__device__ __forceinline__ void philox(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int rnd = 0; rnd < 10; ++rnd) {
    if (rnd) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = (uint32_t)p1;
    c[2] = n2;
    c[3] = (uint32_t)p0;
  }
}

__device__ __forceinline__ double series_log(double x) {
  int e;
  double m = frexp(x, &e);
  if (m < 0.7071067811865476) {
    m = m * 2.0;
    e -= 1;
  }
  const double f = m - 1.0;
  const double s = f / (2.0 + f);
  const double t = s * s;
  double P = 1.0 / 25.0;
#pragma unroll
  for (int k = 11; k >= 0; --k) P = P * t + 1.0 / (double)(2 * k + 1);
  return (double)e * LN2 + 2.0 * s * P;
}

__device__ __forceinline__ double series_exp(double x) {
  if (x < -700.0) return 0.0;
  const double k = rint(x / LN2);
  const double r = (x - k * LN2_HI) - k * LN2_LO;
  // 1 / n!, n = 0..14 (exact integers, correctly rounded quotients)
  constexpr double inv_fact[15] = {1.0 / 1.0, 1.0 / 1.0, 1.0 / 2.0, 1.0 / 6.0, 1.0 / 24.0,
                                   1.0 / 120.0, 1.0 / 720.0, 1.0 / 5040.0, 1.0 / 40320.0,
                                   1.0 / 362880.0, 1.0 / 3628800.0, 1.0 / 39916800.0,
                                   1.0 / 479001600.0, 1.0 / 6227020800.0, 1.0 / 87178291200.0};
  double P = inv_fact[14];
#pragma unroll
  for (int n = 13; n >= 0; --n) P = P * r + inv_fact[n];
  return ldexp(P, (int)k);
}

__device__ __forceinline__ double poly7(const double* c, double r) {
  double v = c[7];
#pragma unroll
  for (int k = 6; k >= 0; --k) v = v * r + c[k];
  return v;
}

__device__ __forceinline__ double inverse_normal(double u) {
  constexpr double PA[8] = {3.3871328727963666080e0, 1.3314166789178437745e+2,
                            1.9715909503065514427e+3, 1.3731693765509461125e+4,
                            4.5921953931549871457e+4, 6.7265770927008700853e+4,
                            3.3430575583588128105e+4, 2.5090809287301226727e+3};
  constexpr double PB[8] = {1.0, 4.2313330701600911252e+1, 6.8718700749205790830e+2,
                            5.3941960214247511077e+3, 2.1213794301586595867e+4,
                            3.9307895800092710610e+4, 2.8729085735721942674e+4,
                            5.2264952788528545610e+3};
  constexpr double PC[8] = {1.42343711074968357734e0, 4.63033784615654529590e0,
                            5.76949722146069140550e0, 3.64784832476320460504e0,
                            1.27045825245236838258e0, 2.41780725177450611770e-1,
                            2.27238449892691845833e-2, 7.74545014278341407640e-4};
  constexpr double PD[8] = {1.0, 2.05319162663775882187e0, 1.67638483018380384940e0,
                            6.89767334985100004550e-1, 1.48103976427480074590e-1,
                            1.51986665636164571966e-2, 5.47593808499534494600e-4,
                            1.05075007164441684324e-9};
  constexpr double PE[8] = {6.65790464350110377720e0, 5.46378491116411436990e0,
                            1.78482653991729133580e0, 2.96560571828504891230e-1,
                            2.65321895265761230930e-2, 1.24266094738807843860e-3,
                            2.71155556874348757815e-5, 2.01033439929228813265e-7};
  constexpr double PF[8] = {1.0, 5.99832206555887937690e-1, 1.36929880922735805310e-1,
                            1.48753612908506148525e-2, 7.86869131145613259100e-4,
                            1.84631831751005468180e-5, 1.42151175831644588870e-7,
                            2.04426310338993978564e-15};
  const double q = u - 0.5;
  if (fabs(q) <= 0.425) {
    const double r = 0.180625 - q * q;
    return q * poly7(PA, r) / poly7(PB, r);
  }
  const double rr = sqrt(-series_log(q < 0 ? u : 1.0 - u));
  double z;
  if (rr <= 5.0) {
    const double r1 = rr - 1.6;
    z = poly7(PC, r1) / poly7(PD, r1);
  } else {
    const double r2 = rr - 5.0;
    z = poly7(PE, r2) / poly7(PF, r2);
  }
  return q < 0 ? -z : z;
}

// N(0, 1) value of node i (instances.noise)
__device__ __forceinline__ double noise(uint64_t seed, int64_t i) {
  uint32_t c[4] = {(uint32_t)i, (uint32_t)((uint64_t)i >> 32), NOISE_STREAM, 0u};
  philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  const double u =
      ((double)(c[0] >> 5) * 67108864.0 + (double)(c[1] >> 6) + 0.5) * (1.0 / 9007199254740992.0);
  return inverse_normal(u);
}

struct Shape {
  double c[3];
  double r;
};

// The generated region: a box [o, o + e) of the global grid G (per axis); its
// nodes in C order are the handle's nodes (the handle's dims may flatten the
// box, e.g. a z-slab pencil (D0, 1, cp) of the box (D0, D1 / P, D2)).
struct Box {
  Dims G;          // global grid
  int64_t o[3], e[3];
  int64_t nb;      // nodes in the box
};

__device__ __forceinline__ void box_coords(const Box& B, int64_t t, int64_t idx[3]) {
  int64_t rem = t;
  for (int a = B.G.nd - 1; a >= 0; --a) {
    idx[a] = B.o[a] + rem % B.e[a];
    rem /= B.e[a];
  }
}
__device__ __forceinline__ int64_t global_index(const Box& B, const int64_t idx[3]) {
  int64_t g = 0;
  for (int a = 0; a < B.G.nd; ++a) g = g * B.G.d[a] + idx[a];
  return g;
}

// mark the box nodes of one disk / ball (block = shape, threads stride its box)
__global__ void k_paint(const Shape* shapes, Box B, uint8_t* mask) {
  const Shape S = shapes[blockIdx.x];
  const int nd = B.G.nd;
  int64_t lo[3] = {0, 0, 0}, ext[3] = {1, 1, 1};
  int64_t vol = 1;
  for (int a = 0; a < nd; ++a) {
    // the shape's box (instances.synth_image), cut to the generated box
    const int64_t l = max(max((int64_t)0, (int64_t)floor(S.c[a] - S.r)), B.o[a]);
    const int64_t h = min(min(B.G.d[a], (int64_t)ceil(S.c[a] + S.r) + 1), B.o[a] + B.e[a]);
    if (h <= l) return;
    lo[a] = l;
    ext[a] = h - l;
    vol *= ext[a];
  }
  const double r2 = S.r * S.r;
  for (int64_t t = threadIdx.x; t < vol; t += blockDim.x) {
    int64_t rem = t, idx[3] = {0, 0, 0};
    for (int a = nd - 1; a >= 0; --a) {
      idx[a] = lo[a] + rem % ext[a];
      rem /= ext[a];
    }
    double d2 = 0.0;  // axis order, from 0.0 (instances.synth_image)
    for (int a = 0; a < nd; ++a) {
      const double dx = (double)idx[a] - S.c[a];
      d2 = d2 + dx * dx;
    }
    if (d2 <= r2) {
      int64_t loc = 0;
      for (int a = 0; a < nd; ++a) loc = loc * B.e[a] + (idx[a] - B.o[a]);
      mask[loc] = 1;
    }
  }
}

// image of the box nodes (noise counter = global node index)
__global__ void k_image(const uint8_t* mask, Box B, uint64_t seed, double sigma, double* img) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < B.nb;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t idx[3];
    box_coords(B, t, idx);
    img[t] = (mask[t] ? 0.7 : 0.3) + sigma * noise(seed, global_index(B, idx));
  }
}

struct EdgeArgs {
  int off[3];      // direction d (global axes)
  int64_t count;   // d-edges inside the box, C order of the box's direction shape
  double inv2s2, scale, lam;
  int integer;
};

// the d-edges between two box nodes (both ends inside the box)
__global__ void k_edges(const double* img, Box B, EdgeArgs E, double* out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E.count;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = e, ja[3] = {0, 0, 0};
    for (int a = B.G.nd - 1; a >= 0; --a) {
      const int64_t ext = B.e[a] - (E.off[a] < 0 ? -E.off[a] : E.off[a]);
      ja[a] = rem % ext;
      rem /= ext;
    }
    int64_t na = 0, nb = 0;
    for (int a = 0; a < B.G.nd; ++a) {
      const int k = E.off[a];
      na = na * B.e[a] + ja[a] + (k < 0 ? -k : 0);
      nb = nb * B.e[a] + ja[a] + (k >= 0 ? k : 0);
    }
    const double diff = img[na] - img[nb];
    double v = series_exp(-(diff * diff) * E.inv2s2);
    if (E.scale != 1.0) v = v * E.scale;
    out[e] = E.integer ? rint(5.0 * E.lam * v) : E.lam * v;
  }
}

__global__ void k_unaries(double* img, int64_t n, int integer) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double w = 10.0 * (img[i] - 0.5);
    if (integer) w = fmin(fmax(rint(w), -10.0), 10.0);
    img[i] = w;
  }
}

}  // namespace gen
}  // namespace pcb
