// Storage tier of the structured-storage-offloading (SSO) path: direct
// (O_DIRECT, page-cache bypassing) reads and writes of tier files into and
// out of page-locked host buffers (hierarchy.py charges
// these bytes to the `gpu_storage` / `host_storage` links).
//
// The B200 box has no GPUDirect Storage (no nvidia-fs), so the GPU <->
// storage "bypass" link is realised as NVMe -> pinned bounce buffer -> DMA:
// the reads below land in the page-locked buffer the copy engine reads from,
// with no page-cache copy in between.  A request is split into page-aligned
// slices read concurrently by `num_threads` threads (NVMe wants several
// requests in flight).  Offsets, sizes and buffer addresses must be
// multiples of kDirectAlign; callers read an aligned superset and index into
// it.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/grinder_b200.h"
#include "grd_common.h"

using namespace grd;

namespace {

constexpr int64_t kDirectAlign = 4096;
constexpr int64_t kSlice = int64_t{8} << 20;   // bytes per request in flight

bool aligned(int64_t v) { return (v % kDirectAlign) == 0; }

// Split [0, nbytes) into kSlice requests served by nt threads; fn(off, len)
// returns 0 or an errno.
template <class Fn>
int parallel_io(int64_t nbytes, int nt, Fn fn) {
    const int64_t nslices = (nbytes + kSlice - 1) / kSlice;
    if (nt < 1) nt = 1;
    if (nt > nslices) nt = static_cast<int>(nslices);
    std::vector<int> err(static_cast<size_t>(nt), 0);
    auto worker = [&](int t) {
        for (int64_t s = t; s < nslices && !err[t]; s += nt) {
            const int64_t off = s * kSlice;
            const int64_t len = std::min(kSlice, nbytes - off);
            err[t] = fn(off, len);
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(worker, t);
    worker(0);
    for (auto& th : pool) th.join();
    for (int e : err)
        if (e) return e;
    return 0;
}

}  // namespace

extern "C" int64_t grd_direct_alignment(void) { return kDirectAlign; }

extern "C" int grd_direct_open(const char* path, int32_t writable, int64_t size, int32_t* fd_out,
                               int32_t* direct_out) {
    clear_error();
    if (!path || !fd_out) return fail(kErrArg, "direct_open: null argument");
    const int flags = (writable ? (O_RDWR | O_CREAT) : O_RDONLY) | O_CLOEXEC;
    int fd = ::open(path, flags | O_DIRECT, 0644);
    int direct = 1;
    if (fd < 0 && errno == EINVAL) {   // filesystem without O_DIRECT (tmpfs, some overlays)
        fd = ::open(path, flags, 0644);
        direct = 0;
    }
    if (fd < 0) return fail(kErrState, "direct_open(%s): %s", path, std::strerror(errno));
    if (direct_out) *direct_out = direct;
    if (writable && size > 0) {
        if (::ftruncate(fd, static_cast<off_t>(round_up(size, kDirectAlign))) != 0) {
            const int e = errno;
            ::close(fd);
            return fail(kErrState, "direct_open(%s): ftruncate: %s", path, std::strerror(e));
        }
    }
    *fd_out = fd;
    return 0;
}

extern "C" int grd_direct_close(int32_t fd) {
    clear_error();
    if (::close(fd) != 0) return fail(kErrState, "direct_close: %s", std::strerror(errno));
    return 0;
}

extern "C" int grd_direct_read(int32_t fd, int64_t offset, int64_t nbytes, void* dst, int32_t num_threads) {
    clear_error();
    if (nbytes == 0) return 0;
    if (fd < 0 || !dst || nbytes < 0 || !aligned(offset) || !aligned(nbytes) ||
        !aligned(static_cast<int64_t>(reinterpret_cast<uintptr_t>(dst))))
        return fail(kErrArg, "direct_read: offset, size and buffer must be %lld-byte aligned",
                    (long long)kDirectAlign);
    char* base = static_cast<char*>(dst);
    const int e = parallel_io(nbytes, num_threads, [&](int64_t off, int64_t len) {
        int64_t done = 0;
        while (done < len) {
            const ssize_t r = ::pread(fd, base + off + done, static_cast<size_t>(len - done),
                                      static_cast<off_t>(offset + off + done));
            if (r < 0) {
                if (errno == EINTR) continue;
                return errno;
            }
            if (r == 0) {   // past end of file: the rest of the slice reads as zeros
                std::memset(base + off + done, 0, static_cast<size_t>(len - done));
                break;
            }
            done += r;
        }
        return 0;
    });
    if (e) return fail(kErrState, "direct_read: %s", std::strerror(e));
    return 0;
}

extern "C" int grd_direct_write(int32_t fd, int64_t offset, int64_t nbytes, const void* src,
                                int32_t num_threads) {
    clear_error();
    if (nbytes == 0) return 0;
    if (fd < 0 || !src || nbytes < 0 || !aligned(offset) || !aligned(nbytes) ||
        !aligned(static_cast<int64_t>(reinterpret_cast<uintptr_t>(src))))
        return fail(kErrArg, "direct_write: offset, size and buffer must be %lld-byte aligned",
                    (long long)kDirectAlign);
    const char* base = static_cast<const char*>(src);
    const int e = parallel_io(nbytes, num_threads, [&](int64_t off, int64_t len) {
        int64_t done = 0;
        while (done < len) {
            const ssize_t r = ::pwrite(fd, base + off + done, static_cast<size_t>(len - done),
                                       static_cast<off_t>(offset + off + done));
            if (r < 0) {
                if (errno == EINTR) continue;
                return errno;
            }
            done += r;
        }
        return 0;
    });
    if (e) return fail(kErrState, "direct_write: %s", std::strerror(e));
    return 0;
}

// Row-run I/O of the SSO manager's tier files (buffered pread / pwrite: runs
// start at arbitrary record offsets).  Run i covers records
// [first[i], first[i] + count[i]) of `record` bytes each, at file offset
// first[i] * record; the runs are packed back to back in `buf`.  Threads
// take whole runs (contiguous ranges of the run list, balanced by bytes).
extern "C" int grd_file_runs(int32_t fd, int32_t write, int64_t record, const int64_t* first,
                             const int64_t* count, int64_t nruns, void* buf, int32_t num_threads) {
    clear_error();
    if (nruns == 0) return 0;
    if (fd < 0 || record <= 0 || !first || !count || !buf || nruns < 0)
        return fail(kErrArg, "file_runs: bad arguments");
    std::vector<int64_t> at(static_cast<size_t>(nruns) + 1, 0);
    for (int64_t i = 0; i < nruns; ++i) {
        if (first[i] < 0 || count[i] < 0) return fail(kErrArg, "file_runs: negative run");
        at[i + 1] = at[i] + count[i] * record;
    }
    const int64_t total = at[nruns];
    int nt = num_threads > 0 ? num_threads : 1;
    if (total < (int64_t{4} << 20)) nt = 1;
    char* base = static_cast<char*>(buf);
    std::vector<int> err(static_cast<size_t>(nt), 0);
    auto worker = [&](int t) {
        // runs whose packed start falls in this thread's byte share
        const int64_t lo = total * t / nt, hi = total * (t + 1) / nt;
        int64_t i = std::lower_bound(at.begin(), at.end() - 1, lo) - at.begin();
        for (; i < nruns && at[i] < hi && !err[t]; ++i) {
            const int64_t len = at[i + 1] - at[i];
            const off_t off = static_cast<off_t>(first[i] * record);
            int64_t done = 0;
            while (done < len) {
                const ssize_t r = write ? ::pwrite(fd, base + at[i] + done, static_cast<size_t>(len - done), off + done)
                                        : ::pread(fd, base + at[i] + done, static_cast<size_t>(len - done), off + done);
                if (r < 0) {
                    if (errno == EINTR) continue;
                    err[t] = errno;
                    break;
                }
                if (r == 0) {   // read past the end of the file: zeros
                    std::memset(base + at[i] + done, 0, static_cast<size_t>(len - done));
                    break;
                }
                done += r;
            }
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(worker, t);
    worker(0);
    for (auto& th : pool) th.join();
    for (int e : err)
        if (e) return fail(kErrState, "file_runs: %s", std::strerror(e));
    return 0;
}

// Row-run copies between a packed buffer and a memory-mapped tier file (the
// SSO manager's storage objects are mapped: scattered row runs become
// memcpy's into the page cache instead of one pread / pwrite per run; the
// kernel writes the pages back).  Same run convention as grd_file_runs.
extern "C" int grd_mem_runs(void* base, int32_t write, int64_t record, const int64_t* first,
                            const int64_t* count, int64_t nruns, void* buf, int32_t num_threads) {
    clear_error();
    if (nruns == 0) return 0;
    if (!base || record <= 0 || !first || !count || !buf || nruns < 0)
        return fail(kErrArg, "mem_runs: bad arguments");
    std::vector<int64_t> at(static_cast<size_t>(nruns) + 1, 0);
    for (int64_t i = 0; i < nruns; ++i) {
        if (first[i] < 0 || count[i] < 0) return fail(kErrArg, "mem_runs: negative run");
        at[i + 1] = at[i] + count[i] * record;
    }
    char* file = static_cast<char*>(base);
    char* packed = static_cast<char*>(buf);
    const int nt = num_threads > 0 ? num_threads : 1;
#pragma omp parallel for num_threads(nt) schedule(dynamic, 64)
    for (int64_t i = 0; i < nruns; ++i) {
        char* f = file + first[i] * record;
        char* b = packed + at[i];
        const size_t len = static_cast<size_t>(at[i + 1] - at[i]);
        if (write) std::memcpy(f, b, len);
        else std::memcpy(b, f, len);
    }
    return 0;
}
