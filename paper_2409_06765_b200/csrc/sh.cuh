// Real spherical harmonics up to degree 3 in fp32 (3DGS constants and signs, Q22).
// colour c = SH((mu - campos)/||mu - campos||); colour is SH-encoded.
#pragma once

namespace gsb {

__device__ constexpr float kC0 = 0.28209479177387814f;
__device__ constexpr float kC1 = 0.4886025119029199f;
__device__ constexpr float kC2[5] = {1.0925484305920792f, -1.0925484305920792f, 0.31539156525252005f,
                                     -1.0925484305920792f, 0.5462742152960396f};
__device__ constexpr float kC3[7] = {-0.5900435899266435f, 2.890611442640554f, -0.4570457994644658f,
                                     0.3731763325901154f, -0.4570457994644658f, 1.445305721320277f,
                                     -0.5900435899266435f};

template <int DEG>
__device__ __forceinline__ void sh_eval_basis(float x, float y, float z, float* Y) {
    Y[0] = kC0;
    if (DEG >= 1) {
        Y[1] = -kC1 * y;
        Y[2] = kC1 * z;
        Y[3] = -kC1 * x;
    }
    if (DEG >= 2) {
        float xx = x * x, yy = y * y, zz = z * z;
        Y[4] = kC2[0] * x * y;
        Y[5] = kC2[1] * y * z;
        Y[6] = kC2[2] * (2.f * zz - xx - yy);
        Y[7] = kC2[3] * x * z;
        Y[8] = kC2[4] * (xx - yy);
        if (DEG >= 3) {
            Y[9] = kC3[0] * y * (3.f * xx - yy);
            Y[10] = kC3[1] * x * y * z;
            Y[11] = kC3[2] * y * (4.f * zz - xx - yy);
            Y[12] = kC3[3] * z * (2.f * zz - 3.f * xx - 3.f * yy);
            Y[13] = kC3[4] * x * (4.f * zz - xx - yy);
            Y[14] = kC3[5] * z * (xx - yy);
            Y[15] = kC3[6] * x * (xx - 3.f * yy);
        }
    }
}

// v_dir += sum_j (dY_j/d(x,y,z)) * w_j   (polynomial partials; normalisation chained by caller)
template <int DEG>
__device__ __forceinline__ void sh_basis_vjp(float x, float y, float z, const float* w, float& gx, float& gy,
                                             float& gz) {
    if (DEG >= 1) {
        gy += -kC1 * w[1];
        gz += kC1 * w[2];
        gx += -kC1 * w[3];
    }
    if (DEG >= 2) {
        gx += kC2[0] * y * w[4];
        gy += kC2[0] * x * w[4];
        gy += kC2[1] * z * w[5];
        gz += kC2[1] * y * w[5];
        gx += kC2[2] * (-2.f * x) * w[6];
        gy += kC2[2] * (-2.f * y) * w[6];
        gz += kC2[2] * (4.f * z) * w[6];
        gx += kC2[3] * z * w[7];
        gz += kC2[3] * x * w[7];
        gx += kC2[4] * (2.f * x) * w[8];
        gy += kC2[4] * (-2.f * y) * w[8];
        if (DEG >= 3) {
            float xx = x * x, yy = y * y, zz = z * z;
            gx += kC3[0] * (6.f * x * y) * w[9];
            gy += kC3[0] * (3.f * xx - 3.f * yy) * w[9];
            gx += kC3[1] * y * z * w[10];
            gy += kC3[1] * x * z * w[10];
            gz += kC3[1] * x * y * w[10];
            gx += kC3[2] * (-2.f * x * y) * w[11];
            gy += kC3[2] * (4.f * zz - xx - 3.f * yy) * w[11];
            gz += kC3[2] * (8.f * y * z) * w[11];
            gx += kC3[3] * (-6.f * x * z) * w[12];
            gy += kC3[3] * (-6.f * y * z) * w[12];
            gz += kC3[3] * (6.f * zz - 3.f * xx - 3.f * yy) * w[12];
            gx += kC3[4] * (4.f * zz - 3.f * xx - yy) * w[13];
            gy += kC3[4] * (-2.f * x * y) * w[13];
            gz += kC3[4] * (8.f * x * z) * w[13];
            gx += kC3[5] * (2.f * x * z) * w[14];
            gy += kC3[5] * (-2.f * y * z) * w[14];
            gz += kC3[5] * (xx - yy) * w[14];
            gx += kC3[6] * (3.f * xx - 3.f * yy) * w[15];
            gy += kC3[6] * (-6.f * x * y) * w[15];
        }
    }
}

}  // namespace gsb
