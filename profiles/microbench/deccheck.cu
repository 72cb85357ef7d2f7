#include <cstdio>
#include <cstdint>
__device__ __forceinline__ float magic_byte(uint32_t u, uint32_t sel) { return __uint_as_float(__byte_perm(u, 0x4B000000u, sel)); }
__global__ void k(int* bad) {
  for (int b = -128; b < 128; ++b) {
    uint32_t w = ((uint32_t)(uint8_t)(int8_t)b) * 0x01010101u;
    uint32_t u = w ^ 0x80808080u;
    for (int j=0;j<4;++j){ float f = magic_byte(u, 0x7540u|j) - 8388736.0f; if (f != (float)b) atomicAdd(bad,1);}
  }
  for (int n = -8; n < 8; ++n) {
    uint32_t w = ((uint32_t)(n & 0xF)) * 0x11111111u;
    uint32_t v = w ^ 0x88888888u; uint32_t lo = v & 0x0F0F0F0Fu, hi = (v>>4)&0x0F0F0F0Fu;
    for (int j=0;j<4;++j){ float a = magic_byte(lo, 0x7540u|j) - 8388616.0f, c = magic_byte(hi,0x7540u|j)-8388616.0f; if (a != (float)n || c != (float)n) atomicAdd(bad,1);}
  }
}
int main(){int*d;cudaMalloc(&d,4);cudaMemset(d,0,4);k<<<1,1>>>(d);int h;cudaMemcpy(&h,d,4,cudaMemcpyDeviceToHost);printf("bad=%d\n",h);}
