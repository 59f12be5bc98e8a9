#pragma once
// pk2.cuh — packed fp32 pairs for sm_100a (K14).  Blackwell issues
// add / mul / fma on two fp32 lanes per thread in ONE instruction (FADD2 /
// FMUL2 / FFMA2, PTX *.rn.f32x2 on .b64), each lane rounded as its scalar
// counterpart.  The FMA pipe's fp32 rate is unchanged (scripts/micro/ffma2.cu:
// 71.6 TFLOP/s FFMA vs 73.4 FFMA2) but the issue slots halve.  A scalar
// broadcast to both lanes is free (ptxas encodes a .F32 operand).
#include <cstdint>

namespace hjcd {

struct f2 {
    unsigned long long v;
};

__device__ __forceinline__ f2 mk2(float a, float b) {
    f2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ f2 bc2(float a) { return mk2(a, a); }
__device__ __forceinline__ void unpk2(f2 a, float& x, float& y) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a.v));
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
    f2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
    f2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
}
// a * b + c, one rounding per lane
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
    f2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(c.v));
    return r;
}

}  // namespace hjcd
