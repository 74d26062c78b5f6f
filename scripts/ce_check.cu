// Copy-engine concurrency experiment (round 2): 16 "clients", each doing
// H2D 48 MiB then D2H 32 MiB per job, 5 jobs, from registered POSIX shm.
// A: both directions on the client's one stream (the GVM's layout so far);
// B: H2D on a per-client upload stream, D2H on its compute stream (event
// dependency); C: as A but one shared H2D stream and one shared D2H stream.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { std::printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

int main() {
    const int C = 16, J = 5;
    const size_t in = 48u << 20, out = 32u << 20;
    std::vector<void*> h(C), dIn(C), dOut(C);
    for (int c = 0; c < C; ++c) {
        std::string name = "/cecheck." + std::to_string(getpid()) + "." + std::to_string(c);
        int fd = shm_open(name.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
        shm_unlink(name.c_str());
        if (ftruncate(fd, in + out)) return 1;
        h[c] = mmap(nullptr, in + out, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
        close(fd);
        std::memset(h[c], 1, in + out);
        CK(cudaHostRegister(h[c], in + out, cudaHostRegisterPortable | cudaHostRegisterMapped));
        CK(cudaMalloc(&dIn[c], in));
        CK(cudaMalloc(&dOut[c], out));
    }
    std::vector<cudaStream_t> s(C), up(C);
    for (int c = 0; c < C; ++c) {
        CK(cudaStreamCreateWithFlags(&s[c], cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&up[c], cudaStreamNonBlocking));
    }
    cudaStream_t sh_up, sh_dn;
    CK(cudaStreamCreateWithFlags(&sh_up, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&sh_dn, cudaStreamNonBlocking));
    std::vector<cudaEvent_t> ev(C * J);
    for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cudaEvent_t t0, t1;
    CK(cudaEventCreate(&t0));
    CK(cudaEventCreate(&t1));
    for (int mode = 0; mode < 3; ++mode) {
        for (int trial = 0; trial < 2; ++trial) {
            CK(cudaDeviceSynchronize());
            CK(cudaEventRecord(t0, 0));
            for (int c = 0; c < C; ++c) CK(cudaStreamWaitEvent(mode == 2 ? sh_up : s[c], t0, 0));
            if (mode == 1) for (int c = 0; c < C; ++c) CK(cudaStreamWaitEvent(up[c], t0, 0));
            if (mode == 2) CK(cudaStreamWaitEvent(sh_dn, t0, 0));
            for (int j = 0; j < J; ++j)
                for (int c = 0; c < C; ++c) {
                    char* hb = static_cast<char*>(h[c]);
                    cudaEvent_t e = ev[c * J + j];
                    if (mode == 0) {
                        CK(cudaMemcpyAsync(dIn[c], hb, in, cudaMemcpyHostToDevice, s[c]));
                        CK(cudaMemcpyAsync(hb + in, dOut[c], out, cudaMemcpyDeviceToHost, s[c]));
                    } else if (mode == 1) {
                        CK(cudaMemcpyAsync(dIn[c], hb, in, cudaMemcpyHostToDevice, up[c]));
                        CK(cudaEventRecord(e, up[c]));
                        CK(cudaStreamWaitEvent(s[c], e, 0));
                        CK(cudaMemcpyAsync(hb + in, dOut[c], out, cudaMemcpyDeviceToHost, s[c]));
                    } else {
                        CK(cudaMemcpyAsync(dIn[c], hb, in, cudaMemcpyHostToDevice, sh_up));
                        CK(cudaEventRecord(e, sh_up));
                        CK(cudaStreamWaitEvent(sh_dn, e, 0));
                        CK(cudaMemcpyAsync(hb + in, dOut[c], out, cudaMemcpyDeviceToHost, sh_dn));
                    }
                }
            for (int c = 0; c < C; ++c) CK(cudaEventRecord(ev[c * J], s[c]));
            for (int c = 0; c < C; ++c) CK(cudaStreamWaitEvent(0, ev[c * J], 0));
            if (mode == 1) for (int c = 0; c < C; ++c) { CK(cudaEventRecord(ev[c * J + 1], up[c])); CK(cudaStreamWaitEvent(0, ev[c * J + 1], 0)); }
            if (mode == 2) { CK(cudaEventRecord(ev[0], sh_dn)); CK(cudaStreamWaitEvent(0, ev[0], 0)); CK(cudaEventRecord(ev[1], sh_up)); CK(cudaStreamWaitEvent(0, ev[1], 0)); }
            CK(cudaEventRecord(t1, 0));
            CK(cudaEventSynchronize(t1));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, t0, t1));
            const double bytes = double(C) * J * (in + out);
            if (trial) std::printf("mode %d (%s): %.2f ms, %.1f GB/s both directions, %.0f jobs/s\n", mode,
                                   mode == 0 ? "one stream per client" : mode == 1 ? "upload stream + compute stream" : "one shared stream per direction",
                                   ms, bytes / (ms * 1e-3) / 1e9, C * J / (ms * 1e-3));
        }
    }
    return 0;
}
