// Probe (development tool): does a global store leave its line readable from L1?
// Pointer chase over 64 lines: plain loads (L1 after warm-up), loads that bypass L1 (.cg),
// and store-then-load of the same word (the pattern of the sweep kernel's set-member finishes).
#include <cstdio>
#include <cstdint>
__global__ void k(uintptr_t *buf, int mode, long long *out) {
    uintptr_t *p = buf;
    for (int i = 0; i < 64; i++) p = (uintptr_t *)*p;          // warm L1
    long long t0 = clock64();
    for (int i = 0; i < 512; i++) {
        if (mode == 0) { p = (uintptr_t *)*p; }
        else if (mode == 1) { p = (uintptr_t *)__ldcg(p); }
        else if (mode == 2) { uintptr_t nx = (uintptr_t)(buf + ((((p - buf) / 16) + 1) & 63) * 16); *p = nx; p = (uintptr_t *)*(volatile uintptr_t *)p; }
        else if (mode == 3) { uintptr_t nx = (uintptr_t)(buf + ((((p - buf) / 16) + 1) & 63) * 16); uintptr_t w;
                              asm volatile("st.global.b64 [%0], %1;" :: "l"(p), "l"(nx) : "memory");
                              asm volatile("ld.global.ca.b64 %0, [%1];" : "=l"(w) : "l"(p) : "memory"); p = (uintptr_t *)w; }
        else { uintptr_t nx = (uintptr_t)(buf + ((((p - buf) / 16) + 1) & 63) * 16); }
    }
    long long t1 = clock64();
    out[0] = (t1 - t0) / 512; out[1] = (long long)p;
}
__global__ void init(uintptr_t *b) { for (int i = 0; i < 64; i++) b[i * 16] = (uintptr_t)(b + ((i + 1) & 63) * 16); }
int main() {
    uintptr_t *b; long long *o, h[2];
    cudaMalloc(&b, 1 << 16); cudaMalloc(&o, 16);
    const char *nm[] = {"ld chain (L1 after warm-up)", "ld.cg chain (L2)", "st; ld.volatile", "st; ld.ca (same word)", "index math only"};
    for (int m = 0; m < 5; m++) {
        init<<<1, 1>>>(b);
        k<<<1, 1>>>(b, m, o); cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
        printf("%-30s %lld cycles/iter\n", nm[m], h[0]);
    }
    return 0;
}
