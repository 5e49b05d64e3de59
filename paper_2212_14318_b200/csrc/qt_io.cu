// qt_io.cu — QT3 tensor files <-> device CD planes.
//
// The reference's binary format (/root/reference/proj/include/qtensor/tensor_io.hpp:16-20,
// src/tensor_io.cpp:37-103): magic "QT3\0", m, n, p as little-endian u64, then
// m*n*p entries slice-major, each four little-endian doubles (w, x, y, z) —
// i.e. an array of 32-byte records {t1.re, t1.im, t2.re, t2.im}.  The device
// layout is two planes (t1, t2), so reading is a streamed de-interleave:
// pread() into two pinned staging buffers in turn, H2D copy, and a kernel that
// splits each 32-byte record into its two 16-byte plane entries (coalesced
// 16-byte loads/stores, HBM-bound byte work); writing is the reverse.  File
// I/O of chunk j+1 overlaps the copy + kernel of chunk j.  Round trips are
// bit-exact (pure byte moves).  Header validation and error kinds follow
// parse_tensor (tensor_io.cpp:56-80): bad magic, truncated header/payload,
// dims outside [1, 2^20] or more than 2^40 entries.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <string>

#include "../../include/qtensor_b200.h"
#include "qt_internal.cuh"

namespace qtb {

namespace {

constexpr size_t kHeader = 4 + 3 * 8;
constexpr size_t kEntry = 32;
constexpr uint64_t kMaxDim = 1ULL << 20;
constexpr uint64_t kMaxEntries = 1ULL << 40;
constexpr size_t kChunkEntries = size_t(1) << 21;  // 64 MB of records per chunk
const unsigned char kMagic[4] = {0x51, 0x54, 0x33, 0x00};

uint64_t le64(const unsigned char* p) {
  uint64_t v = 0;
  for (int k = 0; k < 8; ++k) v |= (uint64_t)p[k] << (8 * k);
  return v;
}
void put_le64(unsigned char* p, uint64_t v) {
  for (int k = 0; k < 8; ++k) p[k] = (unsigned char)(v >> (8 * k));
}

__global__ void deinterleave_kernel(const double2* __restrict__ rec, double2* __restrict__ t1,
                                    double2* __restrict__ t2, uint64_t count) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < count; k += (uint64_t)gridDim.x * blockDim.x) {
    const double2 a = __ldg(&rec[2 * k]);
    const double2 b = __ldg(&rec[2 * k + 1]);
    t1[k] = a;
    t2[k] = b;
  }
}

__global__ void interleave_kernel(const double2* __restrict__ t1, const double2* __restrict__ t2,
                                  double2* __restrict__ rec, uint64_t count) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < count; k += (uint64_t)gridDim.x * blockDim.x) {
    rec[2 * k] = __ldg(&t1[k]);
    rec[2 * k + 1] = __ldg(&t2[k]);
  }
}

unsigned grid_for(uint64_t count) { return (unsigned)std::min<uint64_t>((count + 255) / 256, 148ull * 8); }

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) close(fd);
  }
};

bool pread_all(int fd, void* buf, size_t len, off_t off) {
  char* p = (char*)buf;
  while (len) {
    const ssize_t r = pread(fd, p, len, off);
    if (r <= 0) return false;
    p += r;
    len -= (size_t)r;
    off += r;
  }
  return true;
}

bool pwrite_all(int fd, const void* buf, size_t len, off_t off) {
  const char* p = (const char*)buf;
  while (len) {
    const ssize_t r = pwrite(fd, p, len, off);
    if (r <= 0) return false;
    p += r;
    len -= (size_t)r;
    off += r;
  }
  return true;
}

// Header checks of parse_tensor (tensor_io.cpp:56-74) against the file size.
int check_header(int fd, uint64_t* m, uint64_t* n, uint64_t* p, std::string* err) {
  struct stat st;
  if (fstat(fd, &st) != 0) { *err = "cannot stat"; return QT_EIO; }
  const uint64_t size = (uint64_t)st.st_size;
  unsigned char h[kHeader] = {};
  const size_t got = (size_t)std::min<uint64_t>(size, kHeader);
  if (got && !pread_all(fd, h, got, 0)) { *err = "read failed"; return QT_EIO; }
  if (size < kHeader) {
    if (size < 4 || memcmp(h, kMagic, 4) != 0) { *err = "bad magic"; return QT_EBADMAGIC; }
    *err = "truncated header";
    return QT_ETRUNCATED;
  }
  if (memcmp(h, kMagic, 4) != 0) { *err = "bad magic"; return QT_EBADMAGIC; }
  *m = le64(h + 4);
  *n = le64(h + 12);
  *p = le64(h + 20);
  if (*m == 0 || *n == 0 || *p == 0 || *m > kMaxDim || *n > kMaxDim || *p > kMaxDim || *m * *n > kMaxEntries ||
      *m * *n * *p > kMaxEntries) {
    *err = "dim overflow";
    return QT_EDIMOVERFLOW;
  }
  if (size != kHeader + *m * *n * *p * kEntry) {
    *err = "truncated payload: header dims inconsistent with length";
    return QT_ETRUNCATED;
  }
  return QT_OK;
}

}  // namespace

int qt3_probe(const char* path, uint64_t* m, uint64_t* n, uint64_t* p, std::string* err) {
  Fd f;
  f.fd = open(path, O_RDONLY);
  if (f.fd < 0) { *err = std::string("cannot open for reading: ") + path; return QT_EIO; }
  return check_header(f.fd, m, n, p, err);
}

int qt3_read_device(const char* path, double* t1, double* t2, uint64_t m, uint64_t n, uint64_t p,
                    cudaStream_t stream, std::string* err) {
  Fd f;
  f.fd = open(path, O_RDONLY);
  if (f.fd < 0) { *err = std::string("cannot open for reading: ") + path; return QT_EIO; }
  uint64_t fm = 0, fn = 0, fp = 0;
  int rc = check_header(f.fd, &fm, &fn, &fp, err);
  if (rc) return rc;
  if (fm != m || fn != n || fp != p) { *err = "file dims differ from the destination planes"; return QT_EINVAL; }
  const uint64_t count = m * n * p;
  const size_t chunk = (size_t)std::min<uint64_t>(count, kChunkEntries);
  void* host[2] = {nullptr, nullptr};
  double2* dev = nullptr;
  cudaEvent_t done[2] = {nullptr, nullptr};
  auto cleanup = [&](int code) {
    for (auto& ev : done)
      if (ev) { cudaEventSynchronize(ev); cudaEventDestroy(ev); }
    if (dev) cudaFreeAsync(dev, stream);
    cudaStreamSynchronize(stream);
    for (auto& h : host)
      if (h) cudaFreeHost(h);
    return code;
  };
  for (int b = 0; b < 2; ++b) {
    if (cudaHostAlloc(&host[b], chunk * kEntry, cudaHostAllocDefault) != cudaSuccess) {
      *err = "pinned staging allocation failed";
      return cleanup(QT_ENOMEM);
    }
    cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming);
  }
  if (cudaMallocAsync((void**)&dev, 2 * chunk * kEntry, stream) != cudaSuccess) {
    *err = "device staging allocation failed";
    return cleanup(QT_ENOMEM);
  }
  bool recorded[2] = {false, false};
  for (uint64_t k0 = 0, j = 0; k0 < count; k0 += chunk, ++j) {
    const int b = (int)(j & 1);
    const uint64_t cnt = std::min<uint64_t>(chunk, count - k0);
    if (recorded[b]) cudaEventSynchronize(done[b]);  // staging b free again
    if (!pread_all(f.fd, host[b], cnt * kEntry, (off_t)(kHeader + k0 * kEntry))) {
      *err = "read failed";
      return cleanup(QT_EIO);
    }
    double2* d = dev + 2 * chunk * b;
    cudaError_t e = cudaMemcpyAsync(d, host[b], cnt * kEntry, cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess) {
      deinterleave_kernel<<<grid_for(cnt), 256, 0, stream>>>(d, (double2*)t1 + k0, (double2*)t2 + k0, cnt);
      count_launches(1);
      e = cudaGetLastError();
    }
    if (e != cudaSuccess) { *err = cudaGetErrorString(e); return cleanup(QT_ECUDA); }
    cudaEventRecord(done[b], stream);
    recorded[b] = true;
  }
  return cleanup(QT_OK);
}

int qt3_write_device(const char* path, const double* t1, const double* t2, uint64_t m, uint64_t n, uint64_t p,
                     cudaStream_t stream, std::string* err) {
  if (m == 0 || n == 0 || p == 0) { *err = "zero dims"; return QT_EINVAL; }
  Fd f;
  f.fd = open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (f.fd < 0) { *err = std::string("cannot open for writing: ") + path; return QT_EIO; }
  unsigned char h[kHeader];
  memcpy(h, kMagic, 4);
  put_le64(h + 4, m);
  put_le64(h + 12, n);
  put_le64(h + 20, p);
  if (!pwrite_all(f.fd, h, kHeader, 0)) { *err = "write failed"; return QT_EIO; }
  const uint64_t count = m * n * p;
  const size_t chunk = (size_t)std::min<uint64_t>(count, kChunkEntries);
  void* host[2] = {nullptr, nullptr};
  double2* dev = nullptr;
  cudaEvent_t done[2] = {nullptr, nullptr};
  auto cleanup = [&](int code) {
    for (auto& ev : done)
      if (ev) { cudaEventSynchronize(ev); cudaEventDestroy(ev); }
    if (dev) cudaFreeAsync(dev, stream);
    cudaStreamSynchronize(stream);
    for (auto& hb : host)
      if (hb) cudaFreeHost(hb);
    return code;
  };
  for (int b = 0; b < 2; ++b) {
    if (cudaHostAlloc(&host[b], chunk * kEntry, cudaHostAllocDefault) != cudaSuccess) {
      *err = "pinned staging allocation failed";
      return cleanup(QT_ENOMEM);
    }
    cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming);
  }
  if (cudaMallocAsync((void**)&dev, 2 * chunk * kEntry, stream) != cudaSuccess) {
    *err = "device staging allocation failed";
    return cleanup(QT_ENOMEM);
  }
  // enqueue chunk j+1's interleave + D2H before writing chunk j to the file
  auto enqueue = [&](uint64_t j) -> int {
    const int b = (int)(j & 1);
    const uint64_t k0 = j * chunk, cnt = std::min<uint64_t>(chunk, count - k0);
    double2* d = dev + 2 * chunk * b;
    interleave_kernel<<<grid_for(cnt), 256, 0, stream>>>((const double2*)t1 + k0, (const double2*)t2 + k0, d, cnt);
    count_launches(1);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(host[b], d, cnt * kEntry, cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaEventRecord(done[b], stream);
    if (e != cudaSuccess) { *err = cudaGetErrorString(e); return QT_ECUDA; }
    return QT_OK;
  };
  const uint64_t nchunks = (count + chunk - 1) / chunk;
  int rc = enqueue(0);
  if (rc) return cleanup(rc);
  for (uint64_t j = 0; j < nchunks; ++j) {
    const int b = (int)(j & 1);
    if (j + 1 < nchunks && (rc = enqueue(j + 1))) return cleanup(rc);
    cudaEventSynchronize(done[b]);
    const uint64_t k0 = j * chunk, cnt = std::min<uint64_t>(chunk, count - k0);
    if (!pwrite_all(f.fd, host[b], cnt * kEntry, (off_t)(kHeader + k0 * kEntry))) {
      *err = "write failed";
      return cleanup(QT_EIO);
    }
  }
  return cleanup(QT_OK);
}

}  // namespace qtb
