// GPUDirect Storage probe for the UCPT file path ("pinned
// buffers and/or cuFile GDS"; the reader it would replace is
// /root/reference/pkg/src/ucp/tensor.py:278-320).
//
//   tools/gds_probe PATH [GB]
//
// Writes a GB-sized file at PATH, then reads it back three ways and prints one
// JSON line:
//   - cuFile: cuFileDriverOpen + properties (is nvidia-fs loaded, is the
//     driver in compatibility mode), cuFileHandleRegister on an O_DIRECT fd
//     (falls back to a buffered fd when the file system refuses O_DIRECT),
//     cuFileRead straight into a registered device buffer;
//   - pinned: pread into pinned host memory + cudaMemcpy H2D (what api._pipeline does);
//   - the fs type of PATH (statfs magic).
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/gds_probe.cu -lcufile -o tools/gds_probe
#include <cuda_runtime.h>
#include <cufile.h>
#include <fcntl.h>
#include <sys/statfs.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
  if (argc < 2) {
    fprintf(stderr, "usage: gds_probe PATH [GB]\n");
    return 2;
  }
  const char* path = argv[1];
  const size_t gb = argc > 2 ? strtoull(argv[2], nullptr, 10) : 4;
  const size_t bytes = gb << 30, chunk = 64ull << 20;

  // the test file, written with plain buffered I/O
  fprintf(stderr, "gds_probe: writing %zu GB to %s\n", gb, path);
  {
    int fd = open(path, O_CREAT | O_TRUNC | O_WRONLY, 0644);
    if (fd < 0) { perror("open"); return 1; }
    std::vector<char> buf(chunk, 7);
    for (size_t o = 0; o < bytes; o += chunk)
      if (pwrite(fd, buf.data(), chunk, o) != (ssize_t)chunk) { perror("pwrite"); return 1; }
    fsync(fd);
    close(fd);
  }
  struct statfs sf;
  statfs(path, &sf);

  void* dev = nullptr;
  cudaMalloc(&dev, bytes);

  // cuFile
  fprintf(stderr, "gds_probe: cuFileDriverOpen\n");
  CUfileError_t e = cuFileDriverOpen();
  fprintf(stderr, "gds_probe: driver open err=%d\n", (int)e.err);
  int drv_ok = e.err == CU_FILE_SUCCESS;
  CUfileDrvProps_t props;
  memset(&props, 0, sizeof(props));
  int props_ok = drv_ok && cuFileDriverGetProperties(&props).err == CU_FILE_SUCCESS;
  int direct = 1;
  int fd = open(path, O_RDONLY | O_DIRECT);
  if (fd < 0) { direct = 0; fd = open(path, O_RDONLY); }
  CUfileDescr_t d;
  memset(&d, 0, sizeof(d));
  d.handle.fd = fd;
  d.type = CU_FILE_HANDLE_TYPE_OPAQUE_FD;
  CUfileHandle_t fh;
  int reg_err = -1, buf_err = -1;
  double gds_gbs = -1;
  if (drv_ok) {
    CUfileError_t r = cuFileHandleRegister(&fh, &d);
    reg_err = r.err;
    fprintf(stderr, "gds_probe: handle register err=%d (O_DIRECT %d)\n", reg_err, direct);
    if (r.err == CU_FILE_SUCCESS) {
      buf_err = cuFileBufRegister(dev, bytes, 0).err;
      double best = 1e30;
      for (int rep = 0; rep < 3; rep++) {
        double t0 = now();
        size_t got = 0;
        for (size_t o = 0; o < bytes; o += chunk) {
          ssize_t n = cuFileRead(fh, dev, chunk, o, o);
          if (n > 0) got += n;
        }
        cudaDeviceSynchronize();
        double t = now() - t0;
        if (got == bytes && t < best) best = t;
      }
      if (best < 1e30) gds_gbs = bytes / best / 1e9;
      if (buf_err == CU_FILE_SUCCESS) cuFileBufDeregister(dev);
      cuFileHandleDeregister(fh);
    }
  }
  close(fd);

  // pinned host staging: pread + async H2D, two chunks in flight
  fprintf(stderr, "gds_probe: cufile read %.3f GB/s; pinned leg\n", gds_gbs);
  double pin_gbs = -1;
  {
    int f2 = open(path, O_RDONLY);
    char* h = nullptr;
    cudaHostAlloc((void**)&h, 2 * chunk, 0);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t ev[2];
    cudaEventCreate(&ev[0]);
    cudaEventCreate(&ev[1]);
    double best = 1e30;
    for (int rep = 0; rep < 3; rep++) {
      double t0 = now();
      size_t i = 0;
      for (size_t o = 0; o < bytes; o += chunk, i++) {
        char* b = h + (i & 1) * chunk;
        if (i >= 2) cudaEventSynchronize(ev[i & 1]);
        if (pread(f2, b, chunk, o) != (ssize_t)chunk) break;
        cudaMemcpyAsync((char*)dev + o, b, chunk, cudaMemcpyHostToDevice, s);
        cudaEventRecord(ev[i & 1], s);
      }
      cudaStreamSynchronize(s);
      double t = now() - t0;
      if (t < best) best = t;
    }
    pin_gbs = bytes / best / 1e9;
    close(f2);
    cudaFreeHost(h);
  }
  if (drv_ok) cuFileDriverClose();
  cudaFree(dev);
  unlink(path);

  printf("{\"path\": \"%s\", \"fs_magic\": \"0x%lx\", \"bytes\": %zu, \"o_direct\": %d, "
         "\"driver_open_err\": %d, \"props_ok\": %d, \"nvfs_major\": %u, \"nvfs_minor\": %u, "
         "\"dstatusflags\": \"0x%x\", \"dcontrolflags\": \"0x%x\", \"fflags\": \"0x%x\", "
         "\"handle_register_err\": %d, \"buf_register_err\": %d, "
         "\"cufile_read_GBps\": %.3f, \"pinned_pread_h2d_GBps\": %.3f}\n",
         path, (unsigned long)sf.f_type, bytes, direct, (int)e.err, props_ok,
         props.nvfs.major_version, props.nvfs.minor_version, props.nvfs.dstatusflags,
         props.nvfs.dcontrolflags, props.fflags, reg_err, buf_err, gds_gbs, pin_gbs);
  return 0;
}
