// Directory-tier write/read patterns for a 1.2 GB subgroup file (O_DIRECT):
// striped threads vs one thread, O_TRUNC vs fallocate vs in-place overwrite.
//   g++ -O2 -std=c++20 -pthread scripts/dio_bench.cpp -o /tmp/dio && /tmp/dio <dir>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

static void io(int fd, char* buf, size_t len, off_t off, bool wr, size_t chunk) {
    for (size_t done = 0; done < len;) {
        size_t n = std::min(chunk, len - done);
        ssize_t r = wr ? pwrite(fd, buf + done, n, off + done) : pread(fd, buf + done, n, off + done);
        if (r <= 0) { perror("io"); exit(1); }
        done += r;
    }
}

static void striped(int fd, char* buf, size_t len, bool wr, int threads, size_t chunk) {
    if (threads <= 1) { io(fd, buf, len, 0, wr, chunk); return; }
    size_t stripe = ((len + threads - 1) / threads + 4095) / 4096 * 4096;
    std::vector<std::thread> t;
    for (int s = 0; s < threads; ++s) {
        size_t b = stripe * s;
        if (b >= len) break;
        size_t n = std::min(stripe, len - b);
        t.emplace_back([=] { io(fd, buf + b, n, b, wr, chunk); });
    }
    for (auto& x : t) x.join();
}

int main(int argc, char** argv) {
    std::string dir = argc > 1 ? argv[1] : ".";
    const size_t len = 1200001024;  // 4 KiB multiple
    char* buf = nullptr;
    posix_memalign((void**)&buf, 4096, len);
    memset(buf, 0x5a, len);
    struct Case { const char* name; int threads; size_t chunk; int mode; };  // mode 0 trunc, 1 fallocate, 2 overwrite
    Case cases[] = {{"trunc  4thr whole", 4, len, 0}, {"trunc  1thr 16MB ", 1, 16 << 20, 0},
                    {"trunc  4thr 16MB ", 4, 16 << 20, 0}, {"falloc 4thr 16MB ", 4, 16 << 20, 1},
                    {"falloc 1thr 16MB ", 1, 16 << 20, 1}, {"ovrwr  4thr 16MB ", 4, 16 << 20, 2},
                    {"ovrwr  1thr 16MB ", 1, 16 << 20, 2}, {"ovrwr  4thr whole", 4, len, 2}};
    for (auto& c : cases) {
        for (int rep = 0; rep < 3; ++rep) {
            std::string path = dir + "/f" + std::to_string(rep);
            if (c.mode != 2) unlink(path.c_str());
            if (c.mode == 2) {  // make sure it exists at full size
                struct stat st{};
                if (stat(path.c_str(), &st) != 0 || (size_t)st.st_size != len) {
                    int fd = open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC | O_DIRECT, 0644);
                    io(fd, buf, len, 0, true, 16 << 20); fdatasync(fd); close(fd);
                }
            }
            double t0 = now();
            int flags = O_WRONLY | O_CREAT | O_DIRECT | (c.mode == 0 ? O_TRUNC : 0);
            int fd = open(path.c_str(), flags, 0644);
            if (c.mode == 1 && fallocate(fd, 0, 0, len) != 0) perror("fallocate");
            striped(fd, buf, len, true, c.threads, c.chunk);
            fdatasync(fd);
            close(fd);
            double tw = now() - t0;
            t0 = now();
            fd = open(path.c_str(), O_RDONLY | O_DIRECT);
            striped(fd, buf, len, false, c.threads, c.chunk);
            close(fd);
            double tr = now() - t0;
            printf("%s rep %d: write %.2f GB/s  read %.2f GB/s\n", c.name, rep, len / tw / 1e9, len / tr / 1e9);
            fflush(stdout);
        }
    }
    for (int rep = 0; rep < 3; ++rep) unlink((dir + "/f" + std::to_string(rep)).c_str());
}
