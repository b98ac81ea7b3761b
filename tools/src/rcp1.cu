#include <cstdio>
__global__ void k(float* o) {
    float r;
    asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(o[0]));
    o[1] = r;
    o[2] = o[3] * r;
}
int main() {
    float h[4] = {1.0f, 0.f, 0.f, 0.123456789f}, *d;
    cudaMalloc(&d, 16); cudaMemcpy(d, h, 16, cudaMemcpyHostToDevice);
    k<<<1, 1>>>(d); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("rcp.approx(1.0) = %a  exact=%d  T*rcp==T %d\n", h[1], h[1] == 1.0f, h[2] == h[3]);
    return 0;
}
