// Closed-shell B3LYP semi-local part, pointwise, always in f64.
// Reference: deskdft/xc.py:200-306 (constants :200-205, weights :27-30):
//   f = 0.08 LSDA_x + 0.72 B88_x (incl. Slater) + 0.19 VWN_c(RPA) + 0.81 LYP_c,
// returns exc (per particle), vrho = d f / d n, vsigma = d f / d sigma; zero for
// n < 1e-12 after clamping n, sigma >= 0.  __host__ __device__ so the CPU test
// harness evaluates the identical arithmetic.
#pragma once
#include <math.h>

#ifndef HD
#define HD __host__ __device__ __forceinline__
#endif

namespace dftb {

struct XCOut { double exc, vrho, vsigma; };

// The functional is evaluated in three independent parts (the device XC kernel runs them
// on different warps) and combined by xc_combine; b3lyp_point = parts + combine, so every
// caller performs the identical arithmetic.  Inputs are the clamped n >= 1e-12 and sigma.
struct XPart { double f0, v0, f1, v1, w1; };      // Slater + Becke 88
struct VPart { double f2, v2; };                  // VWN (RPA)
struct LPart { double f3, v3, w3; };              // LYP

namespace b3c {
constexpr double kPi_ = 3.14159265358979323846;
constexpr double CX = 0.7385587663820223;        // 3/4 (3/pi)^(1/3)
constexpr double CXS = 0.9305257363491002;       // 3/2 (3/(4 pi))^(1/3)
constexpr double BETA = 0.0042;
constexpr double VA = 0.0310907, VB = 13.0720, VC = 42.7198, VX0 = -0.409286;
constexpr double LA = 0.04918, LB = 0.132, LC = 0.2533, LD = 0.349;
constexpr double CF = 2.871234000188191;         // 0.3 (3 pi^2)^(2/3)
// derived constants, the correctly rounded values of the reference's expressions (xc.py:237-252)
constexpr double VQ = 0.0448998886415768;        // sqrt(4 VC - VB^2)
constexpr double VX0F = 37.537128437796;         // VX0^2 + VB VX0 + VC
constexpr double V2BQ = 582.2731590427809;       // 2 VB / Q
constexpr double VBX0 = -0.14253052416798392;    // VB VX0 / X(x0)
constexpr double V2BXQ = 545.8110641572265;      // 2 (VB + 2 VX0) / Q
constexpr double CBRT_HALF = 0.7937005259840998; // 2^(-1/3)
}  // namespace b3c

HD XPart b3lyp_x(double n, double sigma) {
    using namespace b3c;
    XPart o;
    const double c13 = cbrt(n);
    // Slater exchange (per particle e = -CX n^(1/3))
    const double el = -CX * c13;
    o.f0 = el * n;
    o.v0 = (4.0 / 3.0) * el;
    // Becke 88 on the spin density ns = n/2, sigma_s = sigma/4
    const double ns = 0.5 * n;
    const double t = c13 * CBRT_HALF, t4 = t * t * t * t;   // (n/2)^(1/3) from n^(1/3)
    const double x = 0.5 * sqrt(sigma) / t4;
    const double ash = asinh(x);
    const double den = 1.0 + 6.0 * BETA * x * ash;
    const double dden = 6.0 * BETA * (ash + x / sqrt(1.0 + x * x));
    const double g = CXS + BETA * x * x / den;
    const double dg = BETA * (2.0 * x * den - x * x * dden) / (den * den);
    o.f1 = -2.0 * t4 * g;
    o.v1 = -(4.0 / 3.0) * t * g + t4 * dg * (4.0 / 3.0) * x / ns;
    o.w1 = 0.5 * (-BETA * (2.0 * den - x * dden) / (2.0 * den * den * t4));
    return o;
}

HD VPart b3lyp_vwn(double n) {
    using namespace b3c;
    VPart o;
    const double rs = cbrt(3.0 / (4.0 * kPi_ * n));
    const double y = sqrt(rs);
    const double Xy = rs + VB * y + VC, iXy = 1.0 / Xy;
    const double at = atan(VQ / (2.0 * y + VB));
    const double ym = y - VX0;
    const double ec = VA * (log(y * y * iXy) + V2BQ * at - VBX0 * (log(ym * ym * iXy) + V2BXQ * at));
    const double dec = VA * (2.0 / y - 2.0 * (y + VB) * iXy - VBX0 * (2.0 / ym - 2.0 * (y + VB + VX0) * iXy));
    o.f2 = ec * n;
    o.v2 = ec - (rs / 3.0) * dec / (2.0 * y);
    return o;
}

HD LPart b3lyp_lyp(double n, double sigma) {
    using namespace b3c;
    LPart o;
    const double c13 = cbrt(n);
    const double tt = 1.0 / c13;                   // n^(-1/3)
    const double Xd = 1.0 + LD * tt, iXd = 1.0 / Xd;
    double tt2 = tt * tt, tt4 = tt2 * tt2, tt8 = tt4 * tt4;
    const double om = tt8 * tt2 * tt * exp(-LC * tt) * iXd;  // t^11 e^{-c t} / X
    const double dl = tt * (LC + LD * iXd);
    const double n143 = n * n * n * n * (c13 * c13);           // n^(14/3)
    const double s37 = 3.0 + 7.0 * dl;
    o.f3 = -LA * n * iXd - LA * LB * om * CF * n143 + LA * LB * om * n * n * sigma * s37 / 72.0;
    o.w3 = LA * LB * om * n * n * s37 / 72.0;
    const double tp = -tt / (3.0 * n);
    const double omp = om * tp * (11.0 * c13 - LC - LD * iXd);
    const double dlp = tp * (LC + LD * iXd - LD * LD * tt * (iXd * iXd));
    o.v3 = -LA * iXd + LA * n * LD * tp * (iXd * iXd) -
           LA * LB * CF * (omp * n143 + om * (14.0 / 3.0) * n143 / n) +
           (LA * LB * sigma / 72.0) * (omp * n * n * s37 + 2.0 * n * om * s37 + 7.0 * om * n * n * dlp);
    return o;
}

HD XCOut xc_combine(double n, const XPart &x, const VPart &v, const LPart &l) {
    XCOut o;
    const double ftot = 0.08 * x.f0 + 0.72 * x.f1 + 0.19 * v.f2 + 0.81 * l.f3;
    o.exc = ftot / n;
    o.vrho = 0.08 * x.v0 + 0.72 * x.v1 + 0.19 * v.v2 + 0.81 * l.v3;
    o.vsigma = 0.72 * x.w1 + 0.81 * l.w3;
    return o;
}

// clamp n, sigma >= 0; zero output below n = 1e-12 (xc.py:287-290)
HD bool b3lyp_clamp(double &n, double &sigma) {
    n = fmax(n, 0.0);
    sigma = fmax(sigma, 0.0);
    return n >= 1e-12;
}

HD XCOut b3lyp_point(double n, double sigma) {
    XCOut o{0.0, 0.0, 0.0};
    if (!b3lyp_clamp(n, sigma)) return o;
    return xc_combine(n, b3lyp_x(n, sigma), b3lyp_vwn(n), b3lyp_lyp(n, sigma));
}

}  // namespace dftb
