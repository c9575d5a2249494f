#include "field.cuh"
using namespace dgkr_b200;
extern "C" __global__ void kmul(const Fe* a, const Fe* b, Fe* o) { int i = threadIdx.x; o[i] = fe_mul<Bn254>(a[i], b[i]); }
extern "C" __global__ void kconst(const Fe* a, Fe* o, const __grid_constant__ FoldConst K) { int i = threadIdx.x; o[i] = fe_mul_const_bn254(a[i], K); }
extern "C" __global__ void kadd(const Fe* a, const Fe* b, Fe* o) { int i = threadIdx.x; o[i] = fe_add<Bn254>(a[i], b[i]); }
extern "C" __global__ void kaccmad(const Fe* a, const Fe* b, Acc* o) { int i = threadIdx.x; Acc x = o[i]; acc_mad(x, a[i], b[i]); o[i] = x; }
