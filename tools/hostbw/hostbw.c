// Host memory bandwidth probe for the e2e conversion question: can the host pack
// reference bytes into bits faster than PCIe moves the bytes?  gcc -O3 -mavx2 -pthread
#include <immintrin.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
static uint8_t* B; static uint32_t* W; static size_t N; static int NT;
static double now() { struct timespec t; clock_gettime(CLOCK_MONOTONIC, &t); return t.tv_sec + t.tv_nsec * 1e-9; }
typedef struct { int id, mode; uint64_t acc; } Arg;
static void* work(void* p) {
    Arg* a = (Arg*)p;
    size_t n32 = N / 32, lo = n32 * a->id / NT, hi = n32 * (a->id + 1) / NT;
    uint64_t acc = 0;
    if (a->mode == 0) {  // read
        for (size_t i = lo; i < hi; ++i) { __m256i v = _mm256_load_si256((const __m256i*)(B + 32 * i)); acc += (uint64_t)_mm256_movemask_epi8(v); }
    } else if (a->mode == 1) {  // pack bytes (0/1) -> bits
        for (size_t i = lo; i < hi; ++i) {
            __m256i v = _mm256_load_si256((const __m256i*)(B + 32 * i));
            W[i] = (uint32_t)_mm256_movemask_epi8(_mm256_slli_epi16(v, 7));
        }
    } else {  // unpack bits -> bytes
        const __m256i sh = _mm256_setr_epi8(0,0,0,0,0,0,0,0,1,1,1,1,1,1,1,1,2,2,2,2,2,2,2,2,3,3,3,3,3,3,3,3);
        const __m256i bit = _mm256_set1_epi64x(0x8040201008040201ull);
        for (size_t i = lo; i < hi; ++i) {
            __m256i v = _mm256_shuffle_epi8(_mm256_set1_epi32((int)W[i]), sh);
            v = _mm256_min_epu8(_mm256_and_si256(v, bit), _mm256_set1_epi8(1));
            _mm256_stream_si256((__m256i*)(B + 32 * i), v);
        }
    }
    a->acc = acc;
    return 0;
}
int main(int argc, char** argv) {
    N = (size_t)(argc > 1 ? atof(argv[1]) : 3.4868e9) / 32 * 32;
    B = aligned_alloc(64, N); W = aligned_alloc(64, N / 8);
    for (size_t i = 0; i < N; ++i) B[i] = (uint8_t)((i * 2654435761u) >> 31 & 1);
    memset(W, 0, N / 8);
    int nts[] = {1, 4, 8, 16, 32};
    const char* names[] = {"read", "pack", "unpack"};
    for (int m = 0; m < 3; ++m)
        for (int k = 0; k < 5; ++k) {
            NT = nts[k];
            pthread_t th[64]; Arg a[64];
            double best = 1e9;
            for (int rep = 0; rep < 3; ++rep) {
                double t0 = now();
                for (int i = 0; i < NT; ++i) { a[i].id = i; a[i].mode = m; pthread_create(&th[i], 0, work, &a[i]); }
                for (int i = 0; i < NT; ++i) pthread_join(th[i], 0);
                double t = now() - t0; if (t < best) best = t;
            }
            printf("%-6s threads=%2d  %.1f ms  %.1f GB/s of bytes\n", names[m], NT, best * 1e3, N / best / 1e9);
            fflush(stdout);
        }
    return 0;
}
