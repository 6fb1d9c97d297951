// ==========================================================================================
// bgs_oracle.cpp — plain, slow, obviously-correct CPU oracle for the BlitzGS per-view
// distributed splatting step (arXiv 2605.13794).
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load this library.  It shares no code, header,
// table or constant generator with the CUDA path (paper_2605_13794_b200/csrc); the only
// shared inputs come from synthetic/ (seeded generators, no method arithmetic).
//
// Citation legend: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n.
// Readings of silent / ambiguous passages are numbered R1..R27 as in DESIGN.md §2.
//
// Build: g++ -O2 -std=c++17 -ffp-contract=off -fno-fast-math -shared -fPIC (no -march: x86-64
// SSE2 float arithmetic is IEEE binary32, no FMA contraction).
//
// Precision: decisions that become integers (gate, radius, rect, alpha test, early stop)
// and the forward values are computed in binary32 exactly as written below (north_star
// fixes fp32 pixels; "where floating point decides an integer both sides take that decision
// in the same precision").  Every accumulation (w, gradients, s) is fp64.  The whole forward
// is a template on the scalar type so that a pure-fp64 instantiation exists for the
// finite-difference pins (tests/test_oracle_fd.py).
// ==========================================================================================
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

// Host threads for the per-Gaussian loops (O3, O11) and the per-tile compositing (O8/O9); 1 =
// the plain sequential oracle.  Every thread count gives bit-identical results: the parallel
// loops write per-index outputs only, and each tile's w / a / gradient increments are buffered
// and applied in tile order, i.e. in exactly the sequential order (or_set_threads; bench.py's
// multi-core baseline).
int g_threads = 1;

// ---------------------------------------------------------------------------------------
// Inputs (oracle-private mirrors of what the Python side passes; NOT the ABI structs)
// ---------------------------------------------------------------------------------------
struct Scene {
  int64_t n;
  const float* mean;   // [n][3]
  const float* quat;   // [n][4]  (w,x,y,z), used as given (activations live outside, R13)
  const float* scale;  // [n][3]
  const float* opac;   // [n]
  const float* sh;     // [n][16][3]
  const uint8_t* lod;  // [n]
};
struct Camera {
  float fx, fy, cx, cy;
  int W, H;
  float R[9], t[3], campos[3], near_clip;
};
struct Gate {
  int enabled, l_max;
  double d0;
  int fb_num, fb_den;  // fallback when fb_den*|L| > fb_num*|G|  (19/20, R20)
};

constexpr int TILE = 16;  // 16x16 tiles (vanilla 3DGS; "tile-based")

// 3DGS SH constants (degree 3), "view-dependent color ... spherical harmonics";
// values of the real SH normalisation with 3DGS's sign convention (R1, R2).
const double SHC0 = 0.28209479177387814;
const double SHC1 = 0.4886025119029199;
const double SHC2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                        -1.0925484305920792, 0.5462742152960396};
const double SHC3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                        0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                        -0.5900435899266435};

template <class T> T k(double v) { return static_cast<T>(v); }

// ---------------------------------------------------------------------------------------
// Eq.5 gate with Eq.4 written as a threshold table (reading R18; pinned by
// test_oracle_pins::test_gate_threshold_equals_log_form against the log form of Eq.4).
//   L_v(d) = clamp(round_half_up(log2(d0/d)), 0, L_max);  keep iff l <= L_v(d)
//   <=> l == 0  or  (l <= L_max and d <= d0 * 2^(1/2 - l))
// ---------------------------------------------------------------------------------------
float d2_threshold(double d0, int l) {
  double v = d0 * std::ldexp(std::sqrt(2.0), -l);
  return static_cast<float>(v * v);
}

// ---------------------------------------------------------------------------------------
// Projection result for one Gaussian (PAPER §3.1; EWA as in 3DGS, readings R3-R8)
// ---------------------------------------------------------------------------------------
template <class T>
struct Proj {
  bool valid = false;
  T mx = 0, my = 0;        // mean2d (pixels)
  T A = 0, B = 0, C = 0;   // conic = inverse of dilated 2D covariance
  T depth = 0;             // camera-frame z
  T rgb[3] = {0, 0, 0};
  bool clamped[3] = {false, false, false};
  T opac = 0;
  T thr = 0;               // alpha-test threshold in power space (D3 / R9)
  int radius = 0;
  int rect[4] = {0, 0, 0, 0};   // tile footprint (R5): xmin, ymin, xmax, ymax (tiles, exclusive max)
  int rect3[4] = {0, 0, 0, 0};  // the 3DGS rect it is cut from (validity, brute force)
  double int_margin = 1e30;    // distance of the pre-truncation floats to an integer (FD safety)
};

inline double frac_dist(double v) { return std::fabs(v - std::nearbyint(v)); }

template <class T> T tmin(T a, T b) { return b < a ? b : a; }
template <class T> T tmax(T a, T b) { return a < b ? b : a; }

// SH basis Y_0..Y_15 along unit direction (x,y,z): written term by term.
template <class T>
void sh_basis(T x, T y, T z, T Y[16]) {
  T xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
  Y[0] = k<T>(SHC0);
  Y[1] = -(k<T>(SHC1) * y);
  Y[2] = k<T>(SHC1) * z;
  Y[3] = -(k<T>(SHC1) * x);
  Y[4] = k<T>(SHC2[0]) * xy;
  Y[5] = k<T>(SHC2[1]) * yz;
  Y[6] = k<T>(SHC2[2]) * ((k<T>(2.0) * zz - xx) - yy);
  Y[7] = k<T>(SHC2[3]) * xz;
  Y[8] = k<T>(SHC2[4]) * (xx - yy);
  Y[9] = (k<T>(SHC3[0]) * y) * (k<T>(3.0) * xx - yy);
  Y[10] = (k<T>(SHC3[1]) * xy) * z;
  Y[11] = (k<T>(SHC3[2]) * y) * ((k<T>(4.0) * zz - xx) - yy);
  Y[12] = (k<T>(SHC3[3]) * z) * ((k<T>(2.0) * zz - k<T>(3.0) * xx) - k<T>(3.0) * yy);
  Y[13] = (k<T>(SHC3[4]) * x) * ((k<T>(4.0) * zz - xx) - yy);
  Y[14] = (k<T>(SHC3[5]) * z) * (xx - yy);
  Y[15] = (k<T>(SHC3[6]) * x) * (xx - k<T>(3.0) * yy);
}

template <class T>
T exp_t(T p);
template <> float exp_t<float>(float p) { return static_cast<float>(std::exp(static_cast<double>(p))); }
template <> double exp_t<double>(double p) { return std::exp(p); }

template <class T>
T thr_of(T o);
// -power of Eq.1 on the projected ellipse, power = -1/2 (A dx^2 + C dy^2) - B dx dy (DESIGN.md
// §4.3, reading R9), evaluated in the pinned order both sides use: with hA = A/2, hC = C/2 (exact),
// -power = fma(hC dy, dy, fma(B dx, dy, (hA dx) dx)), every product and fma rounded once (std::fma
// is the correctly rounded IEEE fused multiply-add, the GPU's FFMA)
template <class T>
T neg_power(T A, T B, T C, T dx, T dy) {
  const T hA = k<T>(0.5) * A, hC = k<T>(0.5) * C;
  const T t1 = (hA * dx) * dx;
  return std::fma(hC * dy, dy, std::fma(B * dx, dy, t1));
}

// Natural logarithm in a fixed sequence of IEEE fp64 operations (reading R30, used for
// thr below so that the alpha-cut threshold is the same bits on both sides by construction rather
// than by two libm's agreeing): u = m 2^e, m in [sqrt(2)/2, sqrt(2)) (exact split),
// ln m = 2 atanh(f) with f = (m - 1)/(m + 1) and the odd series sum_{k<12} f^(2k+1)/(2k+1) in
// Horner form; -ffp-contract=off keeps every step one rounded operation.  Pinned against libm's
// log and oracle/simplify.py in tests/test_oracle_pins.py (P17).
double ln_fixed(double u) {
  int e = 0;
  double m = std::frexp(u, &e);  // u = m 2^e, m in [0.5, 1): exact
  m = m * 2.0;
  e -= 1;
  if (m > 1.4142135623730951) {
    m = m * 0.5;
    e += 1;
  }
  const double f = (m - 1.0) / (m + 1.0);
  const double f2 = f * f;
  double p = 1.0 / 23.0;
  for (int k = 10; k >= 0; --k) p = p * f2 + 1.0 / double(2 * k + 1);
  const double lm = (f + f) * p;
  return double(e) * 0.6931471805599453 + lm;
}

// thr = -ln(255 o): alpha = o*G >= 1/255  <=>  power >= thr  (D3; computed in fp64, rounded)
template <> float thr_of<float>(float o) { return static_cast<float>(-ln_fixed(255.0 * static_cast<double>(o))); }
template <> double thr_of<double>(double o) { return -std::log(255.0 * o); }

template <class T>
Proj<T> project_one(const Scene& s, int64_t i, const Camera& cam, bool no_color) {
  Proj<T> p;
  const float* m = s.mean + 3 * i;
  T mx = m[0], my = m[1], mz = m[2];
  const float* R = cam.R;
  // t_c = R mu + t  (world -> camera)
  T tx = ((T(R[0]) * mx + T(R[1]) * my) + T(R[2]) * mz) + T(cam.t[0]);
  T ty = ((T(R[3]) * mx + T(R[4]) * my) + T(R[5]) * mz) + T(cam.t[1]);
  T tz = ((T(R[6]) * mx + T(R[7]) * my) + T(R[8]) * mz) + T(cam.t[2]);
  if (!(tz > T(cam.near_clip))) return p;  // near clip (R7)

  // Sigma = R(q) S S^T R(q)^T  ("learnable rotation and scale")
  const float* q = s.quat + 4 * i;
  T qw = q[0], qx = q[1], qy = q[2], qz = q[3];
  T xx = qx * qx, yy = qy * qy, zz = qz * qz;
  T xy = qx * qy, xz = qx * qz, yz = qy * qz;
  T wx = qw * qx, wy = qw * qy, wz = qw * qz;
  T Rq[3][3] = {{k<T>(1.0) - k<T>(2.0) * (yy + zz), k<T>(2.0) * (xy - wz), k<T>(2.0) * (xz + wy)},
                {k<T>(2.0) * (xy + wz), k<T>(1.0) - k<T>(2.0) * (xx + zz), k<T>(2.0) * (yz - wx)},
                {k<T>(2.0) * (xz - wy), k<T>(2.0) * (yz + wx), k<T>(1.0) - k<T>(2.0) * (xx + yy)}};
  const float* sc = s.scale + 3 * i;
  T M[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) M[a][b] = Rq[a][b] * T(sc[b]);
  T S[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) S[a][b] = (M[a][0] * M[b][0] + M[a][1] * M[b][1]) + M[a][2] * M[b][2];

  // EWA local-affine Jacobian with the +-1.3*tan(FOV/2) clamp generalised to off-centre c (R8)
  T W = T(cam.W), H = T(cam.H), fx = T(cam.fx), fy = T(cam.fy), cx = T(cam.cx), cy = T(cam.cy);
  T tan_fovx = (k<T>(0.5) * W) / fx;
  T tan_fovy = (k<T>(0.5) * H) / fy;
  T lim_xp = (W - cx) / fx + k<T>(0.3) * tan_fovx;
  T lim_xn = cx / fx + k<T>(0.3) * tan_fovx;
  T lim_yp = (H - cy) / fy + k<T>(0.3) * tan_fovy;
  T lim_yn = cy / fy + k<T>(0.3) * tan_fovy;
  T txtz = tx / tz, tytz = ty / tz;
  T ctx = tmin(lim_xp, tmax(-lim_xn, txtz)) * tz;
  T cty = tmin(lim_yp, tmax(-lim_yn, tytz)) * tz;
  T J00 = fx / tz, J02 = -(fx * ctx) / (tz * tz);
  T J11 = fy / tz, J12 = -(fy * cty) / (tz * tz);
  // Tm = J * Rcam (2x3)
  T Tm[2][3];
  for (int c = 0; c < 3; ++c) {
    Tm[0][c] = J00 * T(R[0 + c]) + J02 * T(R[6 + c]);
    Tm[1][c] = J11 * T(R[3 + c]) + J12 * T(R[6 + c]);
  }
  T U[2][3];
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 3; ++c) U[r][c] = (Tm[r][0] * S[0][c] + Tm[r][1] * S[1][c]) + Tm[r][2] * S[2][c];
  T a = (U[0][0] * Tm[0][0] + U[0][1] * Tm[0][1]) + U[0][2] * Tm[0][2];
  T b = (U[0][0] * Tm[1][0] + U[0][1] * Tm[1][1]) + U[0][2] * Tm[1][2];
  T c = (U[1][0] * Tm[1][0] + U[1][1] * Tm[1][1]) + U[1][2] * Tm[1][2];
  a = a + k<T>(0.3);  // 0.3 px^2 low-pass dilation (R3)
  c = c + k<T>(0.3);
  T det = a * c - b * b;
  if (!(det > T(0))) return p;
  p.A = c / det;
  p.B = (-b) / det;
  p.C = a / det;
  p.mx = fx * txtz + cx;  // pixel centre at integer coordinates (R6)
  p.my = fy * tytz + cy;
  T mid = k<T>(0.5) * (a + c);
  T disc = tmax(k<T>(0.1), mid * mid - det);
  T lambda1 = mid + std::sqrt(disc);
  T rf = std::ceil(k<T>(3.0) * std::sqrt(lambda1));
  rf = tmin(rf, k<T>(1048576.0));  // radius capped at 2^20 px (R4)
  int radius = static_cast<int>(rf);
  p.int_margin = frac_dist(double(k<T>(3.0) * std::sqrt(lambda1)));
  // 3DGS tile rect (R5), float clamp before the integer conversion
  int TX = (cam.W + TILE - 1) / TILE, TY = (cam.H + TILE - 1) / TILE;
  T r_ = T(radius);
  T fx0 = (p.mx - r_) / k<T>(16.0);
  T fy0 = (p.my - r_) / k<T>(16.0);
  T fx1 = ((p.mx + r_) + k<T>(15.0)) / k<T>(16.0);
  T fy1 = ((p.my + r_) + k<T>(15.0)) / k<T>(16.0);
  p.rect[0] = static_cast<int>(tmin(T(TX), tmax(T(0), fx0)));
  p.rect[1] = static_cast<int>(tmin(T(TY), tmax(T(0), fy0)));
  p.rect[2] = static_cast<int>(tmin(T(TX), tmax(T(0), fx1)));
  p.rect[3] = static_cast<int>(tmin(T(TY), tmax(T(0), fy1)));
  if ((p.rect[2] - p.rect[0]) * (p.rect[3] - p.rect[1]) == 0) return p;
  for (T v : {fx0, fy0, fx1, fy1}) p.int_margin = std::min(p.int_margin, frac_dist(double(v)));
  p.radius = radius;
  p.depth = tz;
  p.opac = T(s.opac[i]);
  p.thr = thr_of<T>(p.opac);
  // Tile footprint (reading R5): the 3DGS rect cut to the tiles holding pixel centres of the box
  // around the alpha >= 1/255 ellipse {d : d^T Q d <= -2 thr} (half extents sqrt(-2 thr (Q^-1)_xx),
  // sqrt(-2 thr (Q^-1)_yy), widened by 1e-3 relative + 0.01 px so the box holds every pixel whose
  // fp32 cut test passes).  A tile outside it has no pixel where the splat passes the alpha cut,
  // so N(p) of Eq.2 is unchanged at every pixel (pin P1: tiled == brute force over the 3DGS rects).
  for (int c = 0; c < 4; ++c) p.rect3[c] = p.rect[c];
  {
    T kk = k<T>(-2.0) * p.thr;
    T cdet = p.A * p.C - p.B * p.B;
    if (kk > T(0) && cdet > T(0)) {
      T hx = std::sqrt((kk * p.C) / cdet) * k<T>(1.001) + k<T>(0.01);
      T hy = std::sqrt((kk * p.A) / cdet) * k<T>(1.001) + k<T>(0.01);
      int ex0 = static_cast<int>(tmin(T(TX), tmax(T(0), std::floor((p.mx - hx) / k<T>(16.0)))));
      int ey0 = static_cast<int>(tmin(T(TY), tmax(T(0), std::floor((p.my - hy) / k<T>(16.0)))));
      int ex1 = static_cast<int>(tmin(T(TX), tmax(T(0), std::floor((p.mx + hx) / k<T>(16.0)) + k<T>(1.0))));
      int ey1 = static_cast<int>(tmin(T(TY), tmax(T(0), std::floor((p.my + hy) / k<T>(16.0)) + k<T>(1.0))));
      p.rect[0] = std::max(p.rect[0], ex0);
      p.rect[1] = std::max(p.rect[1], ey0);
      p.rect[2] = std::max(p.rect[0], std::min(p.rect[2], ex1));
      p.rect[3] = std::max(p.rect[1], std::min(p.rect[3], ey1));
    } else {  // o <= 1/255: no pixel passes the cut
      p.rect[2] = p.rect[0];
      p.rect[3] = p.rect[1];
    }
  }
  if (!no_color) {
    // view-dependent colour c_i(d), d = (mu - c_v)/|mu - c_v|  (R1 degree 3, R2 clamp)
    T dx = mx - T(cam.campos[0]), dy = my - T(cam.campos[1]), dz = mz - T(cam.campos[2]);
    T len = std::sqrt((dx * dx + dy * dy) + dz * dz);
    T Y[16];
    sh_basis<T>(dx / len, dy / len, dz / len, Y);
    const float* shp = s.sh + 48 * i;
    for (int ch = 0; ch < 3; ++ch) {
      T col = Y[0] * T(shp[ch]);
      for (int kk = 1; kk < 16; ++kk) col = col + Y[kk] * T(shp[3 * kk + ch]);
      col = col + k<T>(0.5);
      if (col < T(0)) {
        p.clamped[ch] = true;
        col = T(0);
      }
      p.rgb[ch] = col;
    }
  }
  p.valid = true;
  return p;
}

// ---------------------------------------------------------------------------------------
// Step state (one view, M simulated ranks)
// ---------------------------------------------------------------------------------------
struct OwnerState {
  int t_begin = 0, t_end = 0;                 // owned tile run [t_begin, t_end)
  std::vector<int64_t> recv;                  // received splats (global ids), src-rank major
  std::vector<std::pair<int, int64_t>> pairs; // sorted (tile, gid)
  std::vector<int64_t> range_lo, range_hi;    // per owned tile
};

template <class T>
struct Step {
  int M = 1;
  int TX = 0, TY = 0, T_ = 0, W = 0, H = 0;
  std::vector<uint8_t> lod_ok, keep;       // per global Gaussian
  std::vector<int64_t> n_lod, n_keep, fallback;  // per rank
  std::vector<Proj<T>> proj;               // per global Gaussian
  std::vector<int32_t> radius;
  std::vector<int32_t> tile_pairs, owner;  // per tile
  std::vector<uint8_t> dest_mask;          // per global Gaussian
  std::vector<int64_t> counts;             // [M][M] src x dst
  std::vector<OwnerState> owners;
  // forward outputs
  std::vector<float> img, t_final;
  std::vector<int32_t> n_contrib;
  std::vector<double> img64;               // fp64 copy of img (pure-fp64 instantiation for FD)
  double margin_thr = 1e30, margin_clamp = 1e30;  // min |power-thr|, min |o G - 0.99| over evaluations
  std::vector<float> et_margin;            // per pixel: min |T(1-alpha) - 1e-4| / 1e-4 over its tests
  std::vector<double> w;                   // per global Gaussian, fp64 sum of alpha*T
  std::vector<uint64_t> w_fixed;           // per global Gaussian, sum of rint(alpha*T*2^24)
  std::vector<uint32_t> a;                 // per global Gaussian, qualifying pixels (R15)
  // backward
  std::vector<double> g2d;                 // [n][9] d/d(mx,my,A,B,C,o,r,g,b), owner-summed
  std::vector<double> d_mean, d_quat, d_scale, d_opac, d_sh;
  int64_t n_pairs_total = 0;
  double t_project = 0, t_route_sort = 0, t_composite = 0, t_project_bwd = 0;  // seconds
};

struct Contrib {
  int64_t gid;
  double alpha, G, T;
  bool clamped;
};

// Increments one tile makes to per-Gaussian accumulators, in the order the sequential loop
// makes them (replayed by apply_tile).
struct TileOut {
  struct Fwd { int64_t gid; double wgt; uint64_t wfix; };
  struct Bwd { int64_t gid; double g[9]; bool clamped; };
  std::vector<Fwd> fwd;
  std::vector<Bwd> bwd;
  double margin_thr = 1e30, margin_clamp = 1e30;
};

template <class T>
void composite_tile_pixels(Step<T>& st, const std::vector<int64_t>& list, int tile, const float* dLdC, bool backward,
                           TileOut& out) {
  int tx = tile % st.TX, ty = tile / st.TX;
  for (int ly = 0; ly < TILE; ++ly)
    for (int lx = 0; lx < TILE; ++lx) {
      int px = tx * TILE + lx, py = ty * TILE + ly;
      if (px >= st.W || py >= st.H) continue;
      T Tr = T(1);
      T Cc[3] = {T(0), T(0), T(0)};
      int last = 0;
      std::vector<Contrib> cl;
      double margin = 1e30;
      for (size_t kk = 0; kk < list.size(); ++kk) {
        const Proj<T>& p = st.proj[list[kk]];
        // Eq.1 evaluated on the projected ellipse: power = -1/2 d^T Sigma'^-1 d
        T dx = p.mx - T(px), dy = p.my - T(py);
        T power = -neg_power<T>(p.A, p.B, p.C, dx, dy);
        if (power > T(0)) continue;
        out.margin_thr = std::min(out.margin_thr, std::fabs(double(power) - double(p.thr)));
        if (power < p.thr) continue;  // alpha < 1/255 (R9, D3)
        T G = exp_t<T>(power);
        T og = p.opac * G;
        out.margin_clamp = std::min(out.margin_clamp, std::fabs(double(og) - 0.99));
        bool clamped = og > k<T>(0.99);
        T alpha = tmin(k<T>(0.99), og);
        T test_T = Tr * (k<T>(1.0) - alpha);
        margin = std::min(margin, std::fabs(double(test_T) - 1e-4) / 1e-4);
        if (test_T < k<T>(0.0001)) break;  // early termination excludes this splat (R10)
        T wgt = alpha * Tr;
        for (int ch = 0; ch < 3; ++ch) Cc[ch] = Cc[ch] + p.rgb[ch] * wgt;  // Eq.2
        int64_t g = list[kk];
        // w += alpha T (fp64), w_fixed += rint(alpha T 2^24), a += 1 (R15, R29)
        out.fwd.push_back({g, double(wgt), static_cast<uint64_t>(std::rint(double(wgt) * 16777216.0))});
        cl.push_back({g, double(alpha), double(G), double(Tr), clamped});
        Tr = test_T;
        last = int(kk) + 1;
      }
      size_t pix = size_t(py) * st.W + px;
      for (int ch = 0; ch < 3; ++ch) {
        st.img[size_t(ch) * st.W * st.H + pix] = float(Cc[ch]);
        st.img64[size_t(ch) * st.W * st.H + pix] = double(Cc[ch]);
      }
      st.t_final[pix] = float(Tr);
      st.n_contrib[pix] = last;
      st.et_margin[pix] = float(std::min(margin, 1e30));
      if (!dLdC || !backward) continue;
      // backward of Eq.2 ("gradients propagate through both the rasterizer ..."), fp64
      double dL[3] = {dLdC[0 * size_t(st.W) * st.H + pix], dLdC[1 * size_t(st.W) * st.H + pix],
                      dLdC[2 * size_t(st.W) * st.H + pix]};
      double acc[3] = {0, 0, 0};
      for (size_t j = cl.size(); j-- > 0;) {
        const Contrib& c = cl[j];
        const Proj<T>& p = st.proj[c.gid];
        TileOut::Bwd b{c.gid, {0, 0, 0, 0, 0, 0, 0, 0, 0}, c.clamped};
        double* g = b.g;
        double dLda = 0;
        for (int ch = 0; ch < 3; ++ch) {
          g[6 + ch] = c.alpha * c.T * dL[ch];
          dLda += (double(p.rgb[ch]) - acc[ch]) * dL[ch];
        }
        dLda *= c.T;
        for (int ch = 0; ch < 3; ++ch) acc[ch] = c.alpha * double(p.rgb[ch]) + (1.0 - c.alpha) * acc[ch];
        if (!c.clamped) {  // alpha = 0.99 constant: true derivative is zero (R14)
          double o = double(p.opac);
          g[5] = c.G * dLda;
          double dLdpow = c.G * o * dLda;
          double dx = double(p.mx) - px, dy = double(p.my) - py;
          double A = double(p.A), B = double(p.B), C = double(p.C);
          g[0] = dLdpow * (-(A * dx + B * dy));
          g[1] = dLdpow * (-(C * dy + B * dx));
          g[2] = dLdpow * (-0.5 * dx * dx);
          g[3] = dLdpow * (-dx * dy);
          g[4] = dLdpow * (-0.5 * dy * dy);
        }
        out.bwd.push_back(b);
      }
    }
}

// The tile's increments, in the sequential loop's order (per pixel: forward terms front to
// back, then the backward terms back to front; a clamped contributor adds its colour terms only).
template <class T>
void apply_tile(Step<T>& st, const TileOut& out, std::vector<double>* g2d_owner) {
  st.margin_thr = std::min(st.margin_thr, out.margin_thr);
  st.margin_clamp = std::min(st.margin_clamp, out.margin_clamp);
  for (const auto& f : out.fwd) {
    st.w[f.gid] += f.wgt;
    st.w_fixed[f.gid] += f.wfix;
    st.a[f.gid] += 1;
  }
  if (!g2d_owner) return;
  for (const auto& b : out.bwd) {
    double* g = &(*g2d_owner)[9 * b.gid];
    for (int ch = 0; ch < 3; ++ch) g[6 + ch] += b.g[6 + ch];
    if (b.clamped) continue;
    g[5] += b.g[5];
    for (int k = 0; k < 5; ++k) g[k] += b.g[k];
  }
}

// Backward of the projection (a11) in fp64, recomputing from the parameters.
void project_bwd_one(const Scene& s, int64_t i, const Camera& cam, const double* g, const bool clamped[3],
                     double* dmean, double* dquat, double* dscale, double* dopac, double* dsh) {
  const float* m = s.mean + 3 * i;
  double mu[3] = {m[0], m[1], m[2]};
  double R[9];
  for (int j = 0; j < 9; ++j) R[j] = cam.R[j];
  double t_c[3];
  for (int r = 0; r < 3; ++r) t_c[r] = R[3 * r] * mu[0] + R[3 * r + 1] * mu[1] + R[3 * r + 2] * mu[2] + cam.t[r];
  double x = t_c[0], y = t_c[1], z = t_c[2];
  const float* q = s.quat + 4 * i;
  double w = q[0], qx = q[1], qy = q[2], qz = q[3];
  double Rq[3][3] = {{1 - 2 * (qy * qy + qz * qz), 2 * (qx * qy - w * qz), 2 * (qx * qz + w * qy)},
                     {2 * (qx * qy + w * qz), 1 - 2 * (qx * qx + qz * qz), 2 * (qy * qz - w * qx)},
                     {2 * (qx * qz - w * qy), 2 * (qy * qz + w * qx), 1 - 2 * (qx * qx + qy * qy)}};
  const float* sc = s.scale + 3 * i;
  double sv[3] = {sc[0], sc[1], sc[2]};
  double M[3][3], S[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) M[a][b] = Rq[a][b] * sv[b];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) S[a][b] = M[a][0] * M[b][0] + M[a][1] * M[b][1] + M[a][2] * M[b][2];
  double fx = cam.fx, fy = cam.fy, W = cam.W, H = cam.H, cx = cam.cx, cy = cam.cy;
  double tan_fovx = 0.5 * W / fx, tan_fovy = 0.5 * H / fy;
  double lim_xp = (W - cx) / fx + 0.3 * tan_fovx, lim_xn = cx / fx + 0.3 * tan_fovx;
  double lim_yp = (H - cy) / fy + 0.3 * tan_fovy, lim_yn = cy / fy + 0.3 * tan_fovy;
  double txtz = x / z, tytz = y / z;
  bool clx = txtz > lim_xp || txtz < -lim_xn;
  bool cly = tytz > lim_yp || tytz < -lim_yn;
  double ctx = std::min(lim_xp, std::max(-lim_xn, txtz)) * z;
  double cty = std::min(lim_yp, std::max(-lim_yn, tytz)) * z;
  double J00 = fx / z, J02 = -fx * ctx / (z * z), J11 = fy / z, J12 = -fy * cty / (z * z);
  double Tm[2][3];
  for (int c = 0; c < 3; ++c) {
    Tm[0][c] = J00 * R[c] + J02 * R[6 + c];
    Tm[1][c] = J11 * R[3 + c] + J12 * R[6 + c];
  }
  double cov[2][2] = {{0, 0}, {0, 0}};
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 2; ++c)
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) cov[r][c] += Tm[r][a] * S[a][b] * Tm[c][b];
  double a_ = cov[0][0] + 0.3, b_ = cov[0][1], c_ = cov[1][1] + 0.3;
  double det = a_ * c_ - b_ * b_;
  double Q[2][2] = {{c_ / det, -b_ / det}, {-b_ / det, a_ / det}};
  // conic -> dilated cov2d: dL/dS = -Q G_Q Q, G_Q = [[gA, gB/2],[gB/2, gC]]
  double GQ[2][2] = {{g[2], 0.5 * g[3]}, {0.5 * g[3], g[4]}};
  double tmp[2][2], Hs[2][2];
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 2; ++c) tmp[r][c] = Q[r][0] * GQ[0][c] + Q[r][1] * GQ[1][c];
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 2; ++c) Hs[r][c] = -(tmp[r][0] * Q[0][c] + tmp[r][1] * Q[1][c]);
  // symmetric matrix gradient of cov2d (entries a, b(both off-diagonals), c)
  double Gc[2][2] = {{Hs[0][0], 0.5 * (Hs[0][1] + Hs[1][0])}, {0.5 * (Hs[0][1] + Hs[1][0]), Hs[1][1]}};
  // cov2d = Tm S Tm^T: dL/dS3 = Tm^T Gc Tm; dL/dTm = 2 Gc Tm S
  double dS[3][3], dT[2][3];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double v = 0;
      for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 2; ++c) v += Tm[r][a] * Gc[r][c] * Tm[c][b];
      dS[a][b] = v;
    }
  for (int r = 0; r < 2; ++r)
    for (int b = 0; b < 3; ++b) {
      double v = 0;
      for (int c = 0; c < 2; ++c)
        for (int a = 0; a < 3; ++a) v += Gc[r][c] * Tm[c][a] * S[a][b];
      dT[r][b] = 2 * v;
    }
  // Tm = J Rcam: dL/dJ = dL/dTm Rcam^T  (only the 4 non-zero J entries matter)
  double dJ00 = 0, dJ02 = 0, dJ11 = 0, dJ12 = 0;
  for (int c = 0; c < 3; ++c) {
    dJ00 += dT[0][c] * R[c];
    dJ02 += dT[0][c] * R[6 + c];
    dJ11 += dT[1][c] * R[3 + c];
    dJ12 += dT[1][c] * R[6 + c];
  }
  double dx_ = 0, dy_ = 0, dz_ = 0;
  dz_ += dJ00 * (-fx / (z * z)) + dJ11 * (-fy / (z * z));
  dz_ += dJ02 * (2 * fx * ctx / (z * z * z)) + dJ12 * (2 * fy * cty / (z * z * z));
  double dctx = dJ02 * (-fx / (z * z)), dcty = dJ12 * (-fy / (z * z));
  // ctx = clamp(x/z)*z: unclamped -> d/dx = 1; clamped -> d/dz = +-lim (true derivative, R8)
  if (!clx) dx_ += dctx;
  else dz_ += dctx * (txtz > lim_xp ? lim_xp : -lim_xn);
  if (!cly) dy_ += dcty;
  else dz_ += dcty * (tytz > lim_yp ? lim_yp : -lim_yn);
  // mean2d = (fx x/z + cx, fy y/z + cy)
  dx_ += g[0] * fx / z;
  dz_ += -g[0] * fx * x / (z * z);
  dy_ += g[1] * fy / z;
  dz_ += -g[1] * fy * y / (z * z);
  double dtc[3] = {dx_, dy_, dz_};
  for (int c = 0; c < 3; ++c) dmean[c] = R[c] * dtc[0] + R[3 + c] * dtc[1] + R[6 + c] * dtc[2];
  // Sigma = M M^T: dL/dM = 2 dS M (dS symmetric)
  double dM[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double v = 0;
      for (int c = 0; c < 3; ++c) v += (dS[a][c] + dS[c][a]) * M[c][b];
      dM[a][b] = v;
    }
  double dRq[3][3];
  for (int j = 0; j < 3; ++j) {
    dscale[j] = 0;
    for (int r = 0; r < 3; ++r) {
      dscale[j] += Rq[r][j] * dM[r][j];
      dRq[r][j] = dM[r][j] * sv[j];
    }
  }
  // d R(q) / d q (standard unit-quaternion rotation matrix, used as written)
  double gw = 0, gx = 0, gy = 0, gz = 0;
  gy += dRq[0][0] * (-4 * qy); gz += dRq[0][0] * (-4 * qz);
  gx += dRq[0][1] * (2 * qy); gy += dRq[0][1] * (2 * qx); gw += dRq[0][1] * (-2 * qz); gz += dRq[0][1] * (-2 * w);
  gx += dRq[0][2] * (2 * qz); gz += dRq[0][2] * (2 * qx); gw += dRq[0][2] * (2 * qy); gy += dRq[0][2] * (2 * w);
  gx += dRq[1][0] * (2 * qy); gy += dRq[1][0] * (2 * qx); gw += dRq[1][0] * (2 * qz); gz += dRq[1][0] * (2 * w);
  gx += dRq[1][1] * (-4 * qx); gz += dRq[1][1] * (-4 * qz);
  gy += dRq[1][2] * (2 * qz); gz += dRq[1][2] * (2 * qy); gw += dRq[1][2] * (-2 * qx); gx += dRq[1][2] * (-2 * w);
  gx += dRq[2][0] * (2 * qz); gz += dRq[2][0] * (2 * qx); gw += dRq[2][0] * (-2 * qy); gy += dRq[2][0] * (-2 * w);
  gy += dRq[2][1] * (2 * qz); gz += dRq[2][1] * (2 * qy); gw += dRq[2][1] * (2 * qx); gx += dRq[2][1] * (2 * w);
  gx += dRq[2][2] * (-4 * qx); gy += dRq[2][2] * (-4 * qy);
  dquat[0] = gw; dquat[1] = gx; dquat[2] = gy; dquat[3] = gz;
  *dopac = g[5];
  // SH: colour = sum_k Y_k(dir) sh_k + 0.5 (clamped channels pass no gradient)
  double d[3] = {mu[0] - cam.campos[0], mu[1] - cam.campos[1], mu[2] - cam.campos[2]};
  double len = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
  double X = d[0] / len, Yd = d[1] / len, Z = d[2] / len;
  double Y[16];
  sh_basis<double>(X, Yd, Z, Y);
  // dY_k / d(x,y,z)
  double xx = X * X, yy = Yd * Yd, zz = Z * Z;
  double dY[16][3] = {};
  dY[1][1] = -SHC1; dY[2][2] = SHC1; dY[3][0] = -SHC1;
  dY[4][0] = SHC2[0] * Yd; dY[4][1] = SHC2[0] * X;
  dY[5][1] = SHC2[1] * Z; dY[5][2] = SHC2[1] * Yd;
  dY[6][0] = SHC2[2] * (-2 * X); dY[6][1] = SHC2[2] * (-2 * Yd); dY[6][2] = SHC2[2] * (4 * Z);
  dY[7][0] = SHC2[3] * Z; dY[7][2] = SHC2[3] * X;
  dY[8][0] = SHC2[4] * (2 * X); dY[8][1] = SHC2[4] * (-2 * Yd);
  dY[9][0] = SHC3[0] * Yd * 6 * X; dY[9][1] = SHC3[0] * (3 * xx - 3 * yy);
  dY[10][0] = SHC3[1] * Yd * Z; dY[10][1] = SHC3[1] * X * Z; dY[10][2] = SHC3[1] * X * Yd;
  dY[11][0] = SHC3[2] * Yd * (-2 * X); dY[11][1] = SHC3[2] * (4 * zz - xx - 3 * yy); dY[11][2] = SHC3[2] * Yd * 8 * Z;
  dY[12][0] = SHC3[3] * Z * (-6 * X); dY[12][1] = SHC3[3] * Z * (-6 * Yd); dY[12][2] = SHC3[3] * (6 * zz - 3 * xx - 3 * yy);
  dY[13][0] = SHC3[4] * (4 * zz - 3 * xx - yy); dY[13][1] = SHC3[4] * X * (-2 * Yd); dY[13][2] = SHC3[4] * X * 8 * Z;
  dY[14][0] = SHC3[5] * Z * 2 * X; dY[14][1] = SHC3[5] * Z * (-2 * Yd); dY[14][2] = SHC3[5] * (xx - yy);
  dY[15][0] = SHC3[6] * (3 * xx - 3 * yy); dY[15][1] = SHC3[6] * X * (-6 * Yd);
  const float* shp = s.sh + 48 * i;
  double ddir[3] = {0, 0, 0};
  for (int ch = 0; ch < 3; ++ch) {
    double dc = clamped[ch] ? 0.0 : g[6 + ch];
    for (int kk = 0; kk < 16; ++kk) {
      dsh[3 * kk + ch] = Y[kk] * dc;
      for (int e = 0; e < 3; ++e) ddir[e] += dc * double(shp[3 * kk + ch]) * dY[kk][e];
    }
  }
  double dot = ddir[0] * X + ddir[1] * Yd + ddir[2] * Z;
  dmean[0] += (ddir[0] - X * dot) / len;
  dmean[1] += (ddir[1] - Yd * dot) / len;
  dmean[2] += (ddir[2] - Z * dot) / len;
}

template <class T>
Step<T>* run_step(const Scene& s, const Camera& cam, const Gate& gate, const uint32_t* cull_global, int M,
                  int flags, const float* dLdC, int tile_stride) {
  using clk = std::chrono::steady_clock;
  auto secs = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); };
  auto t0 = clk::now();
  const bool no_color = flags & 1;
  auto* st = new Step<T>();
  st->M = M;
  st->W = cam.W;
  st->H = cam.H;
  st->TX = (cam.W + TILE - 1) / TILE;
  st->TY = (cam.H + TILE - 1) / TILE;
  st->T_ = st->TX * st->TY;
  const int64_t n = s.n;
  st->lod_ok.assign(n, 0);
  st->keep.assign(n, 0);
  st->n_lod.assign(M, 0);
  st->n_keep.assign(M, 0);
  st->fallback.assign(M, 0);
  st->proj.assign(n, Proj<T>());
  st->radius.assign(n, 0);

  // O1 shard: owner(i) = i mod M, local j = i div M (R23)
  // O2 gate, Eq.4-6, per rank
  float D2[32];
  for (int l = 0; l < 32; ++l) D2[l] = d2_threshold(gate.d0, l);
  std::vector<int64_t> shard_size(M, 0);
  for (int64_t i = 0; i < n; ++i) {
    int m = int(i % M);
    shard_size[m]++;
    int l = s.lod[i];
    float dx = s.mean[3 * i] - cam.campos[0], dy = s.mean[3 * i + 1] - cam.campos[1],
          dz = s.mean[3 * i + 2] - cam.campos[2];
    float d2 = (dx * dx + dy * dy) + dz * dz;
    bool ok = (l <= gate.l_max) && (l == 0 || d2 <= D2[std::min(l, 31)]);
    st->lod_ok[i] = ok;
    st->n_lod[m] += ok;
  }
  for (int m = 0; m < M; ++m)
    st->fallback[m] = (!gate.enabled) || (int64_t(gate.fb_den) * st->n_lod[m] > int64_t(gate.fb_num) * shard_size[m]);
  for (int64_t i = 0; i < n; ++i) {
    int m = int(i % M);
    bool ok = st->fallback[m] ? true : bool(st->lod_ok[i]);
    bool culled = cull_global && ((cull_global[i >> 5] >> (i & 31)) & 1u);
    st->keep[i] = ok && !culled;
    st->n_keep[m] += st->keep[i];
  }
  // O3 project every kept Gaussian ("every GPU projects only its own local Gaussians")
#pragma omp parallel for schedule(dynamic, 4096) num_threads(g_threads) if (g_threads > 1)
  for (int64_t i = 0; i < n; ++i) {
    if (!st->keep[i]) continue;
    st->proj[i] = project_one<T>(s, i, cam, no_color);
    st->radius[i] = st->proj[i].valid ? st->proj[i].radius : 0;
  }
  auto t1 = clk::now();
  st->t_project = secs(t0, t1);
  // O4 cost-aware tile ownership (reading R24 / D6): c_t = pairs_t + 1
  st->tile_pairs.assign(st->T_, 0);
  for (int64_t i = 0; i < n; ++i) {
    const auto& p = st->proj[i];
    if (!p.valid) continue;
    for (int y = p.rect[1]; y < p.rect[3]; ++y)
      for (int x = p.rect[0]; x < p.rect[2]; ++x) st->tile_pairs[y * st->TX + x]++;
  }
  int64_t Csum = 0;
  for (int t = 0; t < st->T_; ++t) Csum += int64_t(st->tile_pairs[t]) + 1;
  st->owner.assign(st->T_, 0);
  int64_t Pt = 0;
  for (int t = 0; t < st->T_; ++t) {
    int64_t ct = int64_t(st->tile_pairs[t]) + 1;
    int64_t o = ((2 * Pt + ct) * M) / (2 * Csum);
    st->owner[t] = int(std::min<int64_t>(M - 1, o));
    Pt += ct;
  }
  st->owners.assign(M, OwnerState());
  for (int m = 0; m < M; ++m) {
    int b = st->T_, e = st->T_;
    for (int t = 0; t < st->T_; ++t)
      if (st->owner[t] == m) { b = t; break; }
    for (int t = st->T_; t-- > 0;)
      if (st->owner[t] == m) { e = t + 1; break; }
    if (b == st->T_) e = b;
    st->owners[m].t_begin = b;
    st->owners[m].t_end = e;
  }
  // O5 route ("routed to whichever GPUs own the tiles it lands on")
  st->dest_mask.assign(n, 0);
  st->counts.assign(size_t(M) * M, 0);
  for (int src = 0; src < M; ++src)
    for (int64_t i = src; i < n; i += M) {
      const auto& p = st->proj[i];
      if (!p.valid) continue;
      uint32_t mask = 0;
      for (int y = p.rect[1]; y < p.rect[3]; ++y)
        for (int x = p.rect[0]; x < p.rect[2]; ++x) mask |= 1u << st->owner[y * st->TX + x];
      st->dest_mask[i] = uint8_t(mask);
      for (int d = 0; d < M; ++d)
        if (mask >> d & 1u) {
          st->counts[size_t(src) * M + d]++;
          st->owners[d].recv.push_back(i);
        }
    }
  // O6 sort per owner by (tile, depth asc, global id asc) (Eq.2 order N(p); R12)
  for (int m = 0; m < M; ++m) {
    OwnerState& os = st->owners[m];
    for (int64_t g : os.recv) {
      const auto& p = st->proj[g];
      for (int y = p.rect[1]; y < p.rect[3]; ++y)
        for (int x = p.rect[0]; x < p.rect[2]; ++x) {
          int t = y * st->TX + x;
          if (t >= os.t_begin && t < os.t_end) os.pairs.emplace_back(t, g);
        }
    }
    std::sort(os.pairs.begin(), os.pairs.end(), [&](const std::pair<int, int64_t>& u, const std::pair<int, int64_t>& v) {
      if (u.first != v.first) return u.first < v.first;
      T du = st->proj[u.second].depth, dv = st->proj[v.second].depth;
      if (du != dv) return du < dv;
      return u.second < v.second;
    });
    st->n_pairs_total += int64_t(os.pairs.size());
    // O7 ranges
    int nt = os.t_end - os.t_begin;
    os.range_lo.assign(nt, 0);
    os.range_hi.assign(nt, 0);
    for (size_t q = 0; q < os.pairs.size(); ++q) {
      int lt = os.pairs[q].first - os.t_begin;
      if (q == 0 || os.pairs[q - 1].first != os.pairs[q].first) os.range_lo[lt] = int64_t(q);
      if (q + 1 == os.pairs.size() || os.pairs[q + 1].first != os.pairs[q].first) os.range_hi[lt] = int64_t(q) + 1;
    }
  }
  auto t2 = clk::now();
  st->t_route_sort = secs(t1, t2);
  // O8/O9 composite (+ backward) per owner, tiles ascending
  const size_t npix = size_t(cam.W) * cam.H;
  st->img.assign(3 * npix, 0.f);
  st->img64.assign(3 * npix, 0.0);
  st->t_final.assign(npix, 1.f);
  st->n_contrib.assign(npix, 0);
  st->et_margin.assign(npix, 1e30f);
  st->w.assign(n, 0.0);
  st->w_fixed.assign(n, 0);
  st->a.assign(n, 0);
  st->g2d.assign(size_t(9) * n, 0.0);
  std::vector<double> g_owner;
  for (int m = 0; m < M; ++m) {
    OwnerState& os = st->owners[m];
    if (dLdC) g_owner.assign(size_t(9) * n, 0.0);
    std::vector<int> tiles;
    for (int t = os.t_begin; t < os.t_end; ++t) {
      if (tile_stride > 1 && t % tile_stride != 0) continue;  // timing samples only (bench.py)
      tiles.push_back(t);
    }
    // blocks of tiles: composited independently (threads), then applied in tile order
    const size_t blk = g_threads > 1 ? size_t(64) * size_t(g_threads) : 1;
    std::vector<TileOut> outs;
    for (size_t b0 = 0; b0 < tiles.size(); b0 += blk) {
      const size_t nb = std::min(blk, tiles.size() - b0);
      outs.assign(nb, TileOut());
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_threads) if (g_threads > 1)
      for (long long q = 0; q < (long long)nb; ++q) {
        const int t = tiles[b0 + size_t(q)];
        const int lt = t - os.t_begin;
        std::vector<int64_t> list;
        for (int64_t e = os.range_lo[lt]; e < os.range_hi[lt]; ++e) list.push_back(os.pairs[e].second);
        composite_tile_pixels<T>(*st, list, t, dLdC, dLdC != nullptr, outs[size_t(q)]);
      }
      for (size_t q = 0; q < nb; ++q) apply_tile<T>(*st, outs[q], dLdC ? &g_owner : nullptr);
    }
    // O10 reverse route: owner partials summed at the source in owner-ascending order
    if (dLdC)
      for (size_t e = 0; e < g_owner.size(); ++e) st->g2d[e] += g_owner[e];
  }
  auto t3 = clk::now();
  st->t_composite = secs(t2, t3);
  // O11 projection backward
  if (dLdC) {
    st->d_mean.assign(3 * n, 0.0);
    st->d_quat.assign(4 * n, 0.0);
    st->d_scale.assign(3 * n, 0.0);
    st->d_opac.assign(n, 0.0);
    st->d_sh.assign(48 * n, 0.0);
#pragma omp parallel for schedule(dynamic, 4096) num_threads(g_threads) if (g_threads > 1)
    for (int64_t i = 0; i < n; ++i) {
      if (!st->proj[i].valid) continue;
      project_bwd_one(s, i, cam, &st->g2d[9 * i], st->proj[i].clamped, &st->d_mean[3 * i], &st->d_quat[4 * i],
                      &st->d_scale[3 * i], &st->d_opac[i], &st->d_sh[48 * i]);
    }
  }
  st->t_project_bwd = secs(t3, clk::now());
  return st;
}

struct Handle {
  int is_f64 = 0;
  std::unique_ptr<Step<float>> f;
  std::unique_ptr<Step<double>> d;
};

template <class V>
int64_t copy_out(const std::vector<V>& v, void* out) {
  if (out) std::memcpy(out, v.data(), v.size() * sizeof(V));
  return int64_t(v.size());
}

template <class T>
int64_t get_field(Step<T>& st, const std::string& name, int rank, void* out) {
  int64_t n = int64_t(st.proj.size());
  if (name == "lod_ok") return copy_out(st.lod_ok, out);
  if (name == "keep") return copy_out(st.keep, out);
  if (name == "n_lod") return copy_out(st.n_lod, out);
  if (name == "n_keep") return copy_out(st.n_keep, out);
  if (name == "fallback") return copy_out(st.fallback, out);
  if (name == "radius") return copy_out(st.radius, out);
  if (name == "tile_pairs") return copy_out(st.tile_pairs, out);
  if (name == "owner") return copy_out(st.owner, out);
  if (name == "dest_mask") return copy_out(st.dest_mask, out);
  if (name == "counts") return copy_out(st.counts, out);
  if (name == "img") return copy_out(st.img, out);
  if (name == "t_final") return copy_out(st.t_final, out);
  if (name == "n_contrib") return copy_out(st.n_contrib, out);
  if (name == "et_margin") return copy_out(st.et_margin, out);
  if (name == "img64") return copy_out(st.img64, out);
  if (name == "margins") {
    double mr = 1e30;
    for (const auto& p : st.proj) if (p.valid) mr = std::min(mr, p.int_margin);
    std::vector<double> v = {st.margin_thr, st.margin_clamp, mr};
    return copy_out(v, out);
  }
  if (name == "w") return copy_out(st.w, out);
  if (name == "w_fixed") return copy_out(st.w_fixed, out);
  if (name == "a") return copy_out(st.a, out);
  if (name == "g2d") return copy_out(st.g2d, out);
  if (name == "d_mean") return copy_out(st.d_mean, out);
  if (name == "d_quat") return copy_out(st.d_quat, out);
  if (name == "d_scale") return copy_out(st.d_scale, out);
  if (name == "d_opac") return copy_out(st.d_opac, out);
  if (name == "d_sh") return copy_out(st.d_sh, out);
  if (name == "phase_seconds") {
    std::vector<double> v = {st.t_project, st.t_route_sort, st.t_composite, st.t_project_bwd};
    return copy_out(v, out);
  }
  if (name == "n_pairs_total") {
    if (out) *static_cast<int64_t*>(out) = st.n_pairs_total;
    return 1;
  }
  // per-Gaussian projected attributes as fp64 [n][k]
  auto per = [&](int kk, auto fn) -> int64_t {
    if (out) {
      double* o = static_cast<double*>(out);
      for (int64_t i = 0; i < n; ++i) fn(st.proj[i], o + kk * i);
    }
    return kk * n;
  };
  if (name == "mean2d") return per(2, [](const Proj<T>& p, double* o) { o[0] = p.mx; o[1] = p.my; });
  if (name == "conic") return per(3, [](const Proj<T>& p, double* o) { o[0] = p.A; o[1] = p.B; o[2] = p.C; });
  if (name == "depth") return per(1, [](const Proj<T>& p, double* o) { o[0] = p.depth; });
  if (name == "rgb") return per(3, [](const Proj<T>& p, double* o) { for (int c = 0; c < 3; ++c) o[c] = p.rgb[c]; });
  if (name == "thr") return per(1, [](const Proj<T>& p, double* o) { o[0] = p.thr; });
  if (name == "rect") {
    if (out) {
      int32_t* o = static_cast<int32_t*>(out);
      for (int64_t i = 0; i < n; ++i)
        for (int c = 0; c < 4; ++c) o[4 * i + c] = st.proj[i].valid ? st.proj[i].rect[c] : 0;
    }
    return 4 * n;
  }
  if (name == "rect3") {
    if (out) {
      int32_t* o = static_cast<int32_t*>(out);
      for (int64_t i = 0; i < n; ++i)
        for (int c = 0; c < 4; ++c) o[4 * i + c] = st.proj[i].valid ? st.proj[i].rect3[c] : 0;
    }
    return 4 * n;
  }
  // per-owner structures
  if (rank < 0 || rank >= st.M) return -1;
  OwnerState& os = st.owners[rank];
  if (name == "tile_range") {
    if (out) { static_cast<int32_t*>(out)[0] = os.t_begin; static_cast<int32_t*>(out)[1] = os.t_end; }
    return 2;
  }
  if (name == "recv") return copy_out(os.recv, out);
  if (name == "pair_tile") {
    if (out) for (size_t q = 0; q < os.pairs.size(); ++q) static_cast<int32_t*>(out)[q] = os.pairs[q].first;
    return int64_t(os.pairs.size());
  }
  if (name == "pair_gid") {
    if (out) for (size_t q = 0; q < os.pairs.size(); ++q) static_cast<int64_t*>(out)[q] = os.pairs[q].second;
    return int64_t(os.pairs.size());
  }
  if (name == "range_lo") return copy_out(os.range_lo, out);
  if (name == "range_hi") return copy_out(os.range_hi, out);
  return -1;
}

}  // namespace

// =========================================================================================
// C entry points (ctypes; test infrastructure only)
// =========================================================================================
extern "C" {

struct or_scene { int64_t n; const float* mean; const float* quat; const float* scale; const float* opac;
                  const float* sh; const uint8_t* lod; };
struct or_camera { float fx, fy, cx, cy; int32_t W, H; float R[9], t[3], campos[3], near_clip; };
struct or_gate { int32_t enabled, l_max; double d0; int32_t fb_num, fb_den; };

// flags: bit0 = NO_COLOR (skip SH), bit1 = fp64 forward (FD pins)
void* or_step(const or_scene* sc, const or_camera* cm, const or_gate* gt, const uint32_t* cull_global, int32_t M,
              int32_t flags, const float* dLdC, int32_t tile_stride) {
  Scene s{sc->n, sc->mean, sc->quat, sc->scale, sc->opac, sc->sh, sc->lod};
  Camera c;
  std::memcpy(&c, cm, sizeof(Camera));
  Gate g{gt->enabled, gt->l_max, gt->d0, gt->fb_num, gt->fb_den};
  auto* h = new Handle();
  if (flags & 2) {
    h->is_f64 = 1;
    h->d.reset(run_step<double>(s, c, g, cull_global, M, flags, dLdC, tile_stride));
  } else {
    h->f.reset(run_step<float>(s, c, g, cull_global, M, flags, dLdC, tile_stride));
  }
  return h;
}

void or_free(void* h) { delete static_cast<Handle*>(h); }

// Host threads for or_step (1 = sequential; results are bit-identical for every count).
// Returns the count in effect (1 when built without OpenMP).
int32_t or_set_threads(int32_t n) {
#ifdef _OPENMP
  g_threads = n < 1 ? 1 : n;
#else
  (void)n;
  g_threads = 1;
#endif
  return g_threads;
}

// Returns the element count of `name` (for rank-specific fields, of owner `rank`), and
// copies the data into `out` when non-null.  -1 for unknown names.
int64_t or_get(void* hv, const char* name, int32_t rank, void* out) {
  Handle* h = static_cast<Handle*>(hv);
  if (h->is_f64) return get_field(*h->d, name, rank, out);
  return get_field(*h->f, name, rank, out);
}

float or_d2_threshold(double d0, int32_t l) { return d2_threshold(d0, l); }

float or_thr(float o) { return thr_of<float>(o); }
double or_ln(double u) { return ln_fixed(u); }

void or_sh_basis(double x, double y, double z, double* Y) { sh_basis<double>(x, y, z, Y); }

// Brute-force Eq.2 per pixel over ALL projected splats sorted by (depth, gid), a splat taken
// for pixel p iff p's tile lies in its rect (pin P1).  Uses the fp32 projection of `h`.
void or_bruteforce(void* hv, float* img, float* t_final, int32_t* n_contrib_all) {
  Handle* h = static_cast<Handle*>(hv);
  Step<float>& st = *h->f;
  std::vector<int64_t> order;
  for (int64_t i = 0; i < int64_t(st.proj.size()); ++i)
    if (st.proj[i].valid) order.push_back(i);
  std::sort(order.begin(), order.end(), [&](int64_t u, int64_t v) {
    if (st.proj[u].depth != st.proj[v].depth) return st.proj[u].depth < st.proj[v].depth;
    return u < v;
  });
  for (int py = 0; py < st.H; ++py)
    for (int px = 0; px < st.W; ++px) {
      int tx = px / TILE, ty = py / TILE;
      float Tr = 1.f, C[3] = {0, 0, 0};
      int cnt = 0;
      for (int64_t g : order) {
        const Proj<float>& p = st.proj[g];
        if (tx < p.rect3[0] || tx >= p.rect3[2] || ty < p.rect3[1] || ty >= p.rect3[3]) continue;
        float dx = p.mx - float(px), dy = p.my - float(py);
        float power = -neg_power<float>(p.A, p.B, p.C, dx, dy);
        if (power > 0.f || power < p.thr) continue;
        float G = static_cast<float>(std::exp(double(power)));
        float alpha = std::min(0.99f, p.opac * G);
        float test_T = Tr * (1.0f - alpha);
        if (test_T < 0.0001f) break;
        float wgt = alpha * Tr;
        for (int c = 0; c < 3; ++c) C[c] = C[c] + p.rgb[c] * wgt;
        Tr = test_T;
        cnt++;
      }
      size_t pix = size_t(py) * st.W + px;
      for (int c = 0; c < 3; ++c) img[size_t(c) * st.W * st.H + pix] = C[c];
      t_final[pix] = Tr;
      n_contrib_all[pix] = cnt;  // number of contributors (not the list position)
    }
}

// O12 importance (Eq.3; c_rad, c_vis, Cull P:132; readings R15-R17):
//   s += w/(a+eps) for a>0 (w = w_fixed 2^-24), c_rad += radius>0, top-99% mass set by
//   (w_fixed desc, gid asc) smallest prefix with num_den[1]*prefix >= num_den[0]*total.
// Inputs are global arrays (gid order).  cull_out: ceil(n/32) words, bit = !in_set.
void or_importance(int64_t n, const int32_t* radius, const uint64_t* w_fixed, const uint32_t* a, int32_t mass_num,
                   int32_t mass_den, double* s, uint32_t* c_rad, uint32_t* c_vis, uint32_t* cull_out,
                   uint8_t* in_set_out) {
  std::vector<int64_t> pop;
  uint64_t total = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (a[i] > 0) s[i] += (double(w_fixed[i]) / 16777216.0) / (double(a[i]) + 1e-8);
    if (radius[i] > 0) c_rad[i] += 1;
    if (w_fixed[i] > 0) {
      pop.push_back(i);
      total += w_fixed[i];
    }
  }
  std::sort(pop.begin(), pop.end(), [&](int64_t u, int64_t v) {
    if (w_fixed[u] != w_fixed[v]) return w_fixed[u] > w_fixed[v];
    return u < v;
  });
  std::vector<uint8_t> in_set(n, 0);
  unsigned __int128 target = (unsigned __int128)total * (unsigned)mass_num;
  unsigned __int128 prefix = 0;
  for (int64_t q = 0; q < int64_t(pop.size()); ++q) {
    if (total == 0) break;
    if (prefix * (unsigned)mass_den >= target) break;
    in_set[pop[q]] = 1;
    prefix += w_fixed[pop[q]];
  }
  int64_t nw = (n + 31) / 32;
  for (int64_t wi = 0; wi < nw; ++wi) cull_out[wi] = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (in_set[i]) c_vis[i] += 1;
    else cull_out[i >> 5] |= 1u << (i & 31);
    if (in_set_out) in_set_out[i] = in_set[i];
  }
}

}  // extern "C"
