// ubench_pipes.cu -- step 0 of the build plan: per-SM throughput
// of the instructions the fused kernel leans on, alone and paired, so the ALU
// ceiling of DESIGN.md is measured rather than guessed.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench scripts/ubench_pipes.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>

#define N_ITER 4096
#define CHAINS 8

template <int OP>
__device__ __forceinline__ void op(uint32_t (&a)[CHAINS], uint32_t k1, uint32_t k2)
{
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
        uint32_t x = a[c];
        k1 = a[(c + 3) % CHAINS];  // varying operands: nothing folds
        if (OP == 0) asm volatile("add.u32 %0, %0, %1;" : "+r"(x) : "r"(k1));                     // IADD
        if (OP == 1) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x) : "r"(k1), "r"(k2));  // LOP3
        if (OP == 2) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(k1), "r"(k2));      // IMAD
        if (OP == 3) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(x) : "r"(k1), "r"(k2));      // FFMA
        if (OP == 4) asm volatile("{.reg .b32 t; min.u16x2 t, %0, %1; min.u16x2 %0, t, %2;}" : "+r"(x) : "r"(k1), "r"(k2));                                                // VIMNMX3.U16x2
        if (OP == 6) asm volatile("{.reg .b32 t; max.u32 t, %0, %1; max.u32 %0, t, %2;}" : "+r"(x) : "r"(k1), "r"(k2));                                                   // VIMNMX3.U32
        if (OP == 7) asm volatile("min.f16x2 %0, %0, %1;" : "+r"(x) : "r"(k1));  // HMNMX2
        if (OP == 8) asm volatile("shfl.sync.bfly.b32 %0, %0, 1, 0x1f, 0xffffffff;" : "+r"(x));                                        // SHFL
        if (OP == 9) asm volatile("prmt.b32 %0, %0, %1, 0x5432;" : "+r"(x) : "r"(k1));            // PRMT
        if (OP == 10) asm volatile("shf.l.wrap.b32 %0, %0, %1, 1;" : "+r"(x) : "r"(k1));          // SHF
        if (OP == 11) { uint32_t y; asm volatile("min.u32 %0, %1, %2;" : "=r"(y) : "r"(x), "r"(k1)); x = y; }  // IMNMX
        if (OP == 12) asm volatile("{.reg .s32 t; add.s32 t, %0, %1; max.s32 %0, t, %2;}" : "+r"(x) : "r"(k1), "r"(k2));                                  // VIADDMNMX
        if (OP == 14) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(x) : "r"(k1));                   // IMAD.HI
        if (OP == 15) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(k1), "r"(k2));      // IMAD.HI + acc
        if (OP == 16) asm volatile("mul.rn.f32 %0, %0, %1;" : "+r"(x) : "r"(k1));                   // FMUL
        if (OP == 17) asm volatile("add.f32 %0, %0, %1;" : "+r"(x) : "r"(k1));                      // FADD
        if (OP == 18) asm volatile("cvt.rn.f16x2.f32 %0, %0, %1;" : "+r"(x) : "r"(k1));             // F2FP.F16.F32.PACK_AB
        if (OP == 19) asm volatile("add.sat.f32 %0, %0, %1;" : "+r"(x) : "r"(k1));                  // FADD.SAT
        if (OP == 20) asm volatile("cvt.rn.bf16x2.f32 %0, %0, %1;" : "+r"(x) : "r"(k1));            // F2FP.BF16.F32.PACK_AB
        if (OP == 13) { int p; asm volatile("{.reg .pred q; setp.lt.s32 q, %1, %2; selp.b32 %0, 1, 0, q;}" : "=r"(p) : "r"(x), "r"(k1)); x += p; }  // ISETP+SEL+IADD
        a[c] = x;
    }
}

template <int OPA, int OPB>
__global__ void bench(uint32_t *out, uint32_t k1, uint32_t k2, long long *cyc)
{
    uint32_t a[CHAINS], b[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
        a[c] = threadIdx.x * 7 + c;
        b[c] = threadIdx.x * 13 + c;
    }
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < N_ITER; ++i) {
        op<OPA>(a, k1, k2);
        if (OPB >= 0) op<OPB>(b, k2, k1);
    }
    __syncthreads();
    long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s ^= a[c] ^ b[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int OPA, int OPB>
void run(const char *name)
{
    uint32_t *out;
    long long *cyc, h;
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&cyc, 8);
    const int threads = 1024;
    bench<OPA, OPB><<<148, threads>>>(out, 0x3c003c00u, 0x00010001u, cyc);
    cudaDeviceSynchronize();
    bench<OPA, OPB><<<148, threads>>>(out, 0x3c003c00u, 0x00010001u, cyc);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    double ops = (double)N_ITER * CHAINS * threads * (OPB >= 0 ? 2 : 1);
    printf("%-28s %8.2f lane-ops/clk/SM  (warp-inst/clk/SM %.2f)\n", name, ops / h, ops / h / 32);
    cudaFree(out);
    cudaFree(cyc);
}

int main()
{
    run<0, -1>("IADD");
    run<1, -1>("LOP3");
    run<2, -1>("IMAD");
    run<3, -1>("FFMA");
    run<4, -1>("VIMNMX3.U16x2");
    run<6, -1>("VIMNMX3.U32");
    run<11, -1>("IMNMX");
    run<12, -1>("VIADDMNMX");
    run<7, -1>("HMNMX2");
    run<8, -1>("SHFL");
    run<9, -1>("PRMT");
    run<10, -1>("SHF");
    run<13, -1>("ISETP+SEL+IADD (3 inst)");
    run<14, -1>("IMAD.HI");
    run<15, -1>("IMAD.HI+acc");
    run<16, -1>("FMUL");
    run<17, -1>("FADD");
    run<14, 1>("IMAD.HI + LOP3");
    run<15, 3>("IMAD.HI+acc + FFMA");
    run<16, 1>("FMUL + LOP3");
    run<17, 1>("FADD + LOP3");
    run<10, 3>("SHF + FFMA");
    run<4, 3>("VIMNMX3.U16x2 + FFMA");
    run<4, 2>("VIMNMX3.U16x2 + IMAD");
    run<4, 1>("VIMNMX3.U16x2 + LOP3");
    run<1, 3>("LOP3 + FFMA");
    run<1, 2>("LOP3 + IMAD");
    run<0, 3>("IADD + FFMA");
    run<7, 1>("HMNMX2 + LOP3");
    run<7, 3>("HMNMX2 + FFMA");
    run<6, 3>("VIMNMX3.U32 + FFMA");
    run<8, 1>("SHFL + LOP3");
    run<18, -1>("F2FP.F16 (cvt f16x2)");
    run<20, -1>("F2FP.BF16 (cvt bf16x2)");
    run<19, -1>("FADD.SAT");
    run<18, 3>("F2FP.F16 + FFMA");
    run<18, 1>("F2FP.F16 + LOP3");
    run<18, 9>("F2FP.F16 + PRMT");
    run<19, 1>("FADD.SAT + LOP3");
    return 0;
}
