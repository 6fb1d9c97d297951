// a11 backward of the projection (bgs_project_bwd).  PAPER.md P:216 "gradients propagate through
// both the rasterizer and the screen-space routing"; "Training optimizes these primitive
// attributes".  Math identical to the oracle's project_bwd_one:
//   conic -> dilated cov2d (dL/dS = -Q G_Q Q), cov2d = T Sigma T^T (T = J Rcam),
//   J -> t_c with the TRUE derivative of the 1.3 tan(fov/2) clamp (R8), mean2d -> t_c,
//   t_c -> mu (Rcam^T), Sigma = M M^T with M = R(q) diag(s) -> ds, dq (R(q) as written, R13),
//   SH colour -> dsh and, through the normalised view direction, -> dmu (R2 clamp mask).
// One thread per projected local record; gradients are accumulated (+=) into the caller's
// parameter-shaped buffers (each local Gaussian has at most one record per view).  The colour's
// direction derivative comes from k_color (the 3x3 Jacobian sum_k sh[k][ch] dY_k/ddir and the clamp
// bits, 48 B per record), so neither kernel here reads the 192-B SH row: k_project_bwd applies the
// direction term with the geometry, k_project_bwd_shg only writes dsh = Y_k dcol.
#include <cstdlib>

#include "bgs_internal.cuh"

namespace bgs {
namespace {

constexpr float SHC1 = 0.4886025119029199f;
__constant__ float SHC2[5] = {1.0925484305920792f, -1.0925484305920792f, 0.31539156525252005f,
                           -1.0925484305920792f, 0.5462742152960396f};
__constant__ float SHC3[7] = {-0.5900435899266435f, 2.890611442640554f, -0.4570457994644658f,
                           0.3731763325901154f, -0.4570457994644658f, 1.445305721320277f,
                           -0.5900435899266435f};

__global__ void __launch_bounds__(128) k_project_bwd(ProjectBwdArgs a) {
  const int64_t f = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (f >= a.F) return;
  const uint32_t i = a.rec_lidx[f];
  const CameraK& cm = a.cam;
  const float4 mo = __ldg(a.mean_opac + i);
  const float4 q4 = __ldg(a.quat + i);
  const float4 s4 = __ldg(a.scale + i);
  const Acc ac = a.acc[f];
  const float* g = ac.g;
  const float* R = cm.R;
  const float x = R[0] * mo.x + R[1] * mo.y + R[2] * mo.z + cm.t[0];
  const float y = R[3] * mo.x + R[4] * mo.y + R[5] * mo.z + cm.t[1];
  const float z = R[6] * mo.x + R[7] * mo.y + R[8] * mo.z + cm.t[2];
  const float w = q4.x, qx = q4.y, qy = q4.z, qz = q4.w;
  const float Rq[3][3] = {{1.f - 2.f * (qy * qy + qz * qz), 2.f * (qx * qy - w * qz), 2.f * (qx * qz + w * qy)},
                          {2.f * (qx * qy + w * qz), 1.f - 2.f * (qx * qx + qz * qz), 2.f * (qy * qz - w * qx)},
                          {2.f * (qx * qz - w * qy), 2.f * (qy * qz + w * qx), 1.f - 2.f * (qx * qx + qy * qy)}};
  const float sv[3] = {s4.x, s4.y, s4.z};
  float M[3][3], S[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) M[r][c] = Rq[r][c] * sv[c];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) S[r][c] = M[r][0] * M[c][0] + M[r][1] * M[c][1] + M[r][2] * M[c][2];
  const float Wf = float(cm.W), Hf = float(cm.H);
  const float tanx = 0.5f * Wf / cm.fx, tany = 0.5f * Hf / cm.fy;
  const float lim_xp = (Wf - cm.cx) / cm.fx + 0.3f * tanx, lim_xn = cm.cx / cm.fx + 0.3f * tanx;
  const float lim_yp = (Hf - cm.cy) / cm.fy + 0.3f * tany, lim_yn = cm.cy / cm.fy + 0.3f * tany;
  const float txtz = x / z, tytz = y / z;
  const bool clx = txtz > lim_xp || txtz < -lim_xn;
  const bool cly = tytz > lim_yp || tytz < -lim_yn;
  const float ctx = fminf(lim_xp, fmaxf(-lim_xn, txtz)) * z;
  const float cty = fminf(lim_yp, fmaxf(-lim_yn, tytz)) * z;
  const float iz = 1.f / z, iz2 = iz * iz;
  const float J00 = cm.fx * iz, J02 = -cm.fx * ctx * iz2, J11 = cm.fy * iz, J12 = -cm.fy * cty * iz2;
  float Tm[2][3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    Tm[0][c] = J00 * R[c] + J02 * R[6 + c];
    Tm[1][c] = J11 * R[3 + c] + J12 * R[6 + c];
  }
  // cov2d = Tm S Tm^T (+0.3 on the diagonal)
  float U[2][3];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) U[r][c] = Tm[r][0] * S[0][c] + Tm[r][1] * S[1][c] + Tm[r][2] * S[2][c];
  const float ca = U[0][0] * Tm[0][0] + U[0][1] * Tm[0][1] + U[0][2] * Tm[0][2] + 0.3f;
  const float cb = U[0][0] * Tm[1][0] + U[0][1] * Tm[1][1] + U[0][2] * Tm[1][2];
  const float cc = U[1][0] * Tm[1][0] + U[1][1] * Tm[1][1] + U[1][2] * Tm[1][2] + 0.3f;
  const float idet = 1.f / (ca * cc - cb * cb);
  const float Q00 = cc * idet, Q01 = -cb * idet, Q11 = ca * idet;
  // raster moments -> dL/d(mean2d, conic): power = -(A dx^2 + C dy^2)/2 - B dx dy, dL/dpower =
  // o gd; the conic is this thread's Q (the record's A, B, C up to rounding)
  const float o = mo.w;
  const float g_mx = -o * (Q00 * g[0] + Q01 * g[1]);
  const float g_my = -o * (Q01 * g[0] + Q11 * g[1]);
  // dL/dS2 = -Q G_Q Q, G_Q = [[gA, gB/2], [gB/2, gC]], gA = -o m_xx/2, gB = -o m_xy, gC = -o m_yy/2
  const float G00 = -0.5f * o * g[2], G01 = -0.5f * o * g[3], G11 = -0.5f * o * g[4];
  const float t00 = Q00 * G00 + Q01 * G01, t01 = Q00 * G01 + Q01 * G11;
  const float t10 = Q01 * G00 + Q11 * G01, t11 = Q01 * G01 + Q11 * G11;
  const float H00 = -(t00 * Q00 + t01 * Q01);
  const float H01 = -(t00 * Q01 + t01 * Q11);
  const float H10 = -(t10 * Q00 + t11 * Q01);
  const float H11 = -(t10 * Q01 + t11 * Q11);
  const float Gc[2][2] = {{H00, 0.5f * (H01 + H10)}, {0.5f * (H01 + H10), H11}};
  // dL/dSigma = Tm^T Gc Tm ; dL/dTm = 2 Gc Tm Sigma
  float GT[2][3];  // Gc * Tm
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) GT[r][c] = Gc[r][0] * Tm[0][c] + Gc[r][1] * Tm[1][c];
  float dS[3][3];
#pragma unroll
  for (int p = 0; p < 3; ++p)
#pragma unroll
    for (int c = 0; c < 3; ++c) dS[p][c] = Tm[0][p] * GT[0][c] + Tm[1][p] * GT[1][c];
  float dT[2][3];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) dT[r][c] = 2.f * (GT[r][0] * S[0][c] + GT[r][1] * S[1][c] + GT[r][2] * S[2][c]);
  float dJ00 = 0.f, dJ02 = 0.f, dJ11 = 0.f, dJ12 = 0.f;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    dJ00 += dT[0][c] * R[c];
    dJ02 += dT[0][c] * R[6 + c];
    dJ11 += dT[1][c] * R[3 + c];
    dJ12 += dT[1][c] * R[6 + c];
  }
  float dx_ = 0.f, dy_ = 0.f, dz_ = 0.f;
  dz_ += -(dJ00 * cm.fx + dJ11 * cm.fy) * iz2;
  dz_ += 2.f * (dJ02 * cm.fx * ctx + dJ12 * cm.fy * cty) * iz2 * iz;
  const float dctx = -dJ02 * cm.fx * iz2, dcty = -dJ12 * cm.fy * iz2;
  if (!clx) dx_ += dctx;
  else dz_ += dctx * (txtz > lim_xp ? lim_xp : -lim_xn);
  if (!cly) dy_ += dcty;
  else dz_ += dcty * (tytz > lim_yp ? lim_yp : -lim_yn);
  dx_ += g_mx * cm.fx * iz;
  dz_ -= g_mx * cm.fx * x * iz2;
  dy_ += g_my * cm.fy * iz;
  dz_ -= g_my * cm.fy * y * iz2;
  float dmu[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) dmu[c] = R[c] * dx_ + R[3 + c] * dy_ + R[6 + c] * dz_;
  // Sigma = M M^T
  float dM[3][3];
#pragma unroll
  for (int p = 0; p < 3; ++p)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      dM[p][c] = (dS[p][0] + dS[0][p]) * M[0][c] + (dS[p][1] + dS[1][p]) * M[1][c] + (dS[p][2] + dS[2][p]) * M[2][c];
  float ds[3], dRq[3][3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    ds[c] = Rq[0][c] * dM[0][c] + Rq[1][c] * dM[1][c] + Rq[2][c] * dM[2][c];
#pragma unroll
    for (int r = 0; r < 3; ++r) dRq[r][c] = dM[r][c] * sv[c];
  }
  float gw = 0.f, gx = 0.f, gy = 0.f, gz = 0.f;
  gy -= 4.f * qy * dRq[0][0]; gz -= 4.f * qz * dRq[0][0];
  gx += 2.f * qy * dRq[0][1]; gy += 2.f * qx * dRq[0][1]; gw -= 2.f * qz * dRq[0][1]; gz -= 2.f * w * dRq[0][1];
  gx += 2.f * qz * dRq[0][2]; gz += 2.f * qx * dRq[0][2]; gw += 2.f * qy * dRq[0][2]; gy += 2.f * w * dRq[0][2];
  gx += 2.f * qy * dRq[1][0]; gy += 2.f * qx * dRq[1][0]; gw += 2.f * qz * dRq[1][0]; gz += 2.f * w * dRq[1][0];
  gx -= 4.f * qx * dRq[1][1]; gz -= 4.f * qz * dRq[1][1];
  gy += 2.f * qz * dRq[1][2]; gz += 2.f * qy * dRq[1][2]; gw -= 2.f * qx * dRq[1][2]; gx -= 2.f * w * dRq[1][2];
  gx += 2.f * qz * dRq[2][0]; gz += 2.f * qx * dRq[2][0]; gw -= 2.f * qy * dRq[2][0]; gy -= 2.f * w * dRq[2][0];
  gy += 2.f * qz * dRq[2][1]; gz += 2.f * qy * dRq[2][1]; gw += 2.f * qx * dRq[2][1]; gx += 2.f * w * dRq[2][1];
  gx -= 4.f * qx * dRq[2][2]; gy -= 4.f * qy * dRq[2][2];

  // colour -> view direction (mu - c_v)/|mu - c_v| -> mu: dL/ddir = sum_ch dcol_ch J[ch], then the
  // normalisation's projection (I - d d^T)/|mu - c_v|
  {
    const float4 j0 = __ldg(a.jdir + 3 * f), j1 = __ldg(a.jdir + 3 * f + 1), j2 = __ldg(a.jdir + 3 * f + 2);
    const uint32_t clamped = __float_as_uint(j2.y);
    const float d0 = (clamped & 1u) ? 0.f : g[6], d1 = (clamped & 2u) ? 0.f : g[7], d2 = (clamped & 4u) ? 0.f : g[8];
    const float gx_ = d0 * j0.x + d1 * j0.w + d2 * j1.z;
    const float gy_ = d0 * j0.y + d1 * j1.x + d2 * j1.w;
    const float gz_ = d0 * j0.z + d1 * j1.y + d2 * j2.x;
    const float ddx = mo.x - cm.campos[0], ddy = mo.y - cm.campos[1], ddz = mo.z - cm.campos[2];
    const float il = 1.f / sqrtf(ddx * ddx + ddy * ddy + ddz * ddz);
    const float X = ddx * il, Y = ddy * il, Z = ddz * il;
    const float dot = gx_ * X + gy_ * Y + gz_ * Z;
    dmu[0] += (gx_ - X * dot) * il;
    dmu[1] += (gy_ - Y * dot) * il;
    dmu[2] += (gz_ - Z * dot) * il;
  }

  // accumulate with 128-bit reductions (no read round trip on the SM; the L2 adds)
  atomicAdd(a.g_mean_opac + i, make_float4(dmu[0], dmu[1], dmu[2], g[5]));
  atomicAdd(a.g_quat + i, make_float4(gw, gx, gy, gz));
  atomicAdd(a.g_scale + i, make_float4(ds[0], ds[1], ds[2], 0.f));
}

// dL/dsh[k][ch] = Y_k(dir) dcol_ch (dcol = 0 on clamped channels, R2).  kT threads per record
// (adjacent lanes), each writing 16 / kT coefficients = 12 / kT float4 of the gradient row with
// 128-bit reductions: no SH row read (k_color's clamp bits decide dcol).
template <int kT>
__global__ void __launch_bounds__(256) k_project_bwd_shg(ProjectBwdArgs a) {
  constexpr int kC = 16 / kT;      // coefficients per thread
  constexpr int kQ = 3 * kC / 4;   // float4 per thread
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t f = t / kT;
  const int h = int(threadIdx.x % kT);
  if (f >= a.F) return;
  const uint32_t i = a.rec_lidx[f];
  const CameraK& cm = a.cam;
  const float4 mo = __ldg(a.mean_opac + i);
  const float* g = a.acc[f].g;
  const uint32_t clamped = __float_as_uint(__ldg(reinterpret_cast<const float*>(a.jdir + 3 * f + 2) + 1));
  const float dcol[3] = {(clamped & 1u) ? 0.f : g[6], (clamped & 2u) ? 0.f : g[7], (clamped & 4u) ? 0.f : g[8]};
  const float ddx = mo.x - cm.campos[0], ddy = mo.y - cm.campos[1], ddz = mo.z - cm.campos[2];
  const float il = 1.f / sqrtf(ddx * ddx + ddy * ddy + ddz * ddz);
  const float X = ddx * il, Y = ddy * il, Z = ddz * il;
  const float xx = X * X, yy = Y * Y, zz = Z * Z, xy = X * Y, yz = Y * Z, xz = X * Z;
  float Yb[kC];
#pragma unroll
  for (int c = 0; c < kC; ++c) {
    const int k = kC * h + c;
    float y0;
    switch (k) {
      case 0: y0 = 0.28209479177387814f; break;
      case 1: y0 = -SHC1 * Y; break;
      case 2: y0 = SHC1 * Z; break;
      case 3: y0 = -SHC1 * X; break;
      case 4: y0 = SHC2[0] * xy; break;
      case 5: y0 = SHC2[1] * yz; break;
      case 6: y0 = SHC2[2] * (2.f * zz - xx - yy); break;
      case 7: y0 = SHC2[3] * xz; break;
      case 8: y0 = SHC2[4] * (xx - yy); break;
      case 9: y0 = SHC3[0] * Y * (3.f * xx - yy); break;
      case 10: y0 = SHC3[1] * xy * Z; break;
      case 11: y0 = SHC3[2] * Y * (4.f * zz - xx - yy); break;
      case 12: y0 = SHC3[3] * Z * (2.f * zz - 3.f * xx - 3.f * yy); break;
      case 13: y0 = SHC3[4] * X * (4.f * zz - xx - yy); break;
      case 14: y0 = SHC3[5] * Z * (xx - yy); break;
      default: y0 = SHC3[6] * X * (xx - 3.f * yy); break;
    }
    Yb[c] = y0;
  }
  float4* gsh = reinterpret_cast<float4*>(a.g_sh + size_t(48) * i) + kQ * h;
#pragma unroll
  for (int k = 0; k < kQ; ++k) {
    const int e = 4 * k;
    atomicAdd(gsh + k, make_float4(Yb[(e) / 3] * dcol[(e) % 3], Yb[(e + 1) / 3] * dcol[(e + 1) % 3],
                                   Yb[(e + 2) / 3] * dcol[(e + 2) % 3], Yb[(e + 3) / 3] * dcol[(e + 3) % 3]));
  }
}

}  // namespace

void launch_project_bwd(const ProjectBwdArgs& a, cudaStream_t s) {
  if (a.F <= 0) return;
  k_project_bwd<<<unsigned((a.F + 127) / 128), 128, 0, s>>>(a);
  k_project_bwd_shg<4><<<unsigned((4 * a.F + 255) / 256), 256, 0, s>>>(a);
}

}  // namespace bgs
