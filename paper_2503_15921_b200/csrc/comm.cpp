// Cross-rank exchange of the selector statistics: one
// communicator per device/process, ncclAllGather of the per-(request, SSM)
// ArmEstimate{sum, count} rows (bandit.hpp:24-39) -- the path's only collective --
// plus the host-side reductions bench.py needs (max of device times over ranks,
// a barrier). NCCL is loaded at first use (dlopen "libnccl.so.2"), so the library
// links no NCCL and shares whichever copy the process already has.
//
// A TCP transport with the same semantics (gather to rank 0 in rank order, then
// broadcast) runs without any GPU: the CPU tests drive the C-ABI gather with it in
// two processes. Both transports return identical, rank-ordered results, so every
// rank derives the same selector input.
#include <arpa/inet.h>
#include <dlfcn.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <sys/socket.h>
#include <unistd.h>

#include <cuda_runtime.h>
#include <nccl.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "spin_c.h"
#include "status.hpp"

namespace spin {
namespace {

struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string why;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return;
    }
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.init_rank = reinterpret_cast<decltype(api.init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.destroy = reinterpret_cast<decltype(api.destroy)>(dlsym(h, "ncclCommDestroy"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    if (!api.get_unique_id || !api.init_rank || !api.destroy || !api.all_gather || !api.all_reduce)
      why = "libnccl.so.2 lacks a required symbol";
  });
  if (!why.empty()) fail(SPIN_IO_ERROR, why);
  return api;
}

void check_nccl(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const NcclApi& a = nccl();
    fail(SPIN_IO_ERROR, std::string(what) + ": " + (a.error_string ? a.error_string(r) : "nccl error"));
  }
}

// ---------------------------------------------------------------- TCP transport
void send_all(int fd, const void* p, size_t n) {
  const char* c = static_cast<const char*>(p);
  while (n > 0) {
    const ssize_t k = ::send(fd, c, n, MSG_NOSIGNAL);
    if (k <= 0) fail(SPIN_IO_ERROR, "comm: send failed");
    c += k, n -= static_cast<size_t>(k);
  }
}
void recv_all(int fd, void* p, size_t n) {
  char* c = static_cast<char*>(p);
  while (n > 0) {
    const ssize_t k = ::recv(fd, c, n, 0);
    if (k <= 0) fail(SPIN_IO_ERROR, "comm: peer closed the connection");
    c += k, n -= static_cast<size_t>(k);
  }
}

bool parse_endpoint(const uint8_t* id, std::string* host, int* port) {
  const std::string s(reinterpret_cast<const char*>(id), strnlen(reinterpret_cast<const char*>(id), 127));
  const size_t colon = s.rfind(':');
  if (colon == std::string::npos) return false;
  *host = s.substr(0, colon);
  *port = std::atoi(s.c_str() + colon + 1);
  return *port > 0 && *port < 65536;
}

}  // namespace

struct Comm {
  int backend = SPIN_COMM_TCP;
  int rank = 0, world = 1, device = 0;
  // NCCL
  ncclComm_t nc = nullptr;
  cudaStream_t stream = nullptr;
  void* dbuf = nullptr;
  size_t dbuf_bytes = 0;
  // TCP: rank 0 holds one socket per peer (index = peer rank), others one to rank 0
  std::vector<int> peers;
  int listen_fd = -1;

  ~Comm() {
    if (nc) nccl().destroy(nc);
    if (dbuf) cudaFree(dbuf);
    if (stream) cudaStreamDestroy(stream);
    for (int fd : peers)
      if (fd >= 0) ::close(fd);
    if (listen_fd >= 0) ::close(listen_fd);
  }

  void* device_buffer(size_t bytes) {
    if (bytes > dbuf_bytes) {
      if (dbuf) cudaFree(dbuf);
      dbuf = nullptr;
      check_cuda(cudaMalloc(&dbuf, bytes), "comm buffer");
      dbuf_bytes = bytes;
    }
    return dbuf;
  }

  // Gathers `bytes` from every rank into out[world * bytes], rank order, on every rank.
  void allgather_bytes(const void* in, void* out, size_t bytes) {
    char* o = static_cast<char*>(out);
    if (backend == SPIN_COMM_NCCL) {
      check_cuda(cudaSetDevice(device), "cudaSetDevice");
      char* d = static_cast<char*>(device_buffer(bytes * (world + 1)));
      check_cuda(cudaMemcpyAsync(d, in, bytes, cudaMemcpyHostToDevice, stream), "h2d");
      check_nccl(nccl().all_gather(d, d + bytes, bytes, ncclChar, nc, stream), "ncclAllGather");
      check_cuda(cudaMemcpyAsync(o, d + bytes, bytes * world, cudaMemcpyDeviceToHost, stream), "d2h");
      check_cuda(cudaStreamSynchronize(stream), "allgather");
      return;
    }
    if (world == 1) {
      std::memcpy(o, in, bytes);
      return;
    }
    if (rank == 0) {
      std::memcpy(o, in, bytes);
      for (int r = 1; r < world; ++r) recv_all(peers[r], o + bytes * r, bytes);
      for (int r = 1; r < world; ++r) send_all(peers[r], o, bytes * world);
    } else {
      send_all(peers[0], in, bytes);
      recv_all(peers[0], o, bytes * world);
    }
  }

  void tcp_connect(const uint8_t* id) {
    std::string host;
    int port = 0;
    if (!parse_endpoint(id, &host, &port)) fail(SPIN_CONFIG_ERROR, "comm: TCP id must hold \"host:port\"");
    sockaddr_in addr{};
    addr.sin_family = AF_INET;
    addr.sin_port = htons(static_cast<uint16_t>(port));
    if (inet_pton(AF_INET, host.c_str(), &addr.sin_addr) != 1) fail(SPIN_CONFIG_ERROR, "comm: bad IPv4 host");
    peers.assign(world, -1);
    if (rank == 0) {
      listen_fd = ::socket(AF_INET, SOCK_STREAM, 0);
      const int one = 1;
      setsockopt(listen_fd, SOL_SOCKET, SO_REUSEADDR, &one, sizeof one);
      if (::bind(listen_fd, reinterpret_cast<sockaddr*>(&addr), sizeof addr) != 0 || ::listen(listen_fd, world) != 0)
        fail(SPIN_IO_ERROR, "comm: rank 0 cannot listen on " + host + ":" + std::to_string(port));
      for (int k = 1; k < world; ++k) {
        const int fd = ::accept(listen_fd, nullptr, nullptr);
        if (fd < 0) fail(SPIN_IO_ERROR, "comm: accept failed");
        setsockopt(fd, IPPROTO_TCP, TCP_NODELAY, &one, sizeof one);
        int32_t peer = -1;
        recv_all(fd, &peer, 4);
        if (peer < 1 || peer >= world || peers[peer] >= 0) fail(SPIN_IO_ERROR, "comm: bad peer rank");
        peers[peer] = fd;
      }
      return;
    }
    const auto deadline = std::chrono::steady_clock::now() + std::chrono::seconds(120);
    for (;;) {
      const int fd = ::socket(AF_INET, SOCK_STREAM, 0);
      if (::connect(fd, reinterpret_cast<sockaddr*>(&addr), sizeof addr) == 0) {
        const int one = 1;
        setsockopt(fd, IPPROTO_TCP, TCP_NODELAY, &one, sizeof one);
        const int32_t me = rank;
        send_all(fd, &me, 4);
        peers[0] = fd;
        return;
      }
      ::close(fd);
      if (std::chrono::steady_clock::now() > deadline) fail(SPIN_IO_ERROR, "comm: cannot reach rank 0");
      std::this_thread::sleep_for(std::chrono::milliseconds(20));
    }
  }
};

}  // namespace spin

using namespace spin;

struct spin_comm {
  Comm c;
};

extern "C" {

spin_status spin_comm_unique_id(int32_t backend, uint8_t* id) {
  return guarded([&] {
    if (!id) fail(SPIN_INPUT_ERROR, "spin_comm_unique_id: null id");
    std::memset(id, 0, SPIN_COMM_ID_BYTES);
    if (backend == SPIN_COMM_NCCL) {
      ncclUniqueId u;
      check_nccl(nccl().get_unique_id(&u), "ncclGetUniqueId");
      static_assert(sizeof(u) == SPIN_COMM_ID_BYTES, "NCCL unique id size");
      std::memcpy(id, &u, sizeof u);
      return;
    }
    if (backend != SPIN_COMM_TCP) fail(SPIN_CONFIG_ERROR, "spin_comm_unique_id: unknown backend");
    // a free loopback port, reserved by bind-and-release
    const int fd = ::socket(AF_INET, SOCK_STREAM, 0);
    sockaddr_in a{};
    a.sin_family = AF_INET;
    a.sin_port = 0;
    inet_pton(AF_INET, "127.0.0.1", &a.sin_addr);
    socklen_t len = sizeof a;
    if (::bind(fd, reinterpret_cast<sockaddr*>(&a), sizeof a) != 0 ||
        getsockname(fd, reinterpret_cast<sockaddr*>(&a), &len) != 0) {
      ::close(fd);
      fail(SPIN_IO_ERROR, "spin_comm_unique_id: no free port");
    }
    const int port = ntohs(a.sin_port);
    ::close(fd);
    std::snprintf(reinterpret_cast<char*>(id), SPIN_COMM_ID_BYTES, "127.0.0.1:%d", port);
  });
}

spin_status spin_comm_create(int32_t backend, int32_t device, int32_t rank, int32_t world, const uint8_t* id,
                             spin_comm** out) {
  return guarded([&] {
    if (!id || !out) fail(SPIN_INPUT_ERROR, "spin_comm_create: null argument");
    if (world < 1 || rank < 0 || rank >= world) fail(SPIN_CONFIG_ERROR, "spin_comm_create: bad rank / world");
    auto cm = std::make_unique<spin_comm>();
    Comm& c = cm->c;
    c.backend = backend, c.rank = rank, c.world = world, c.device = device;
    if (backend == SPIN_COMM_NCCL) {
      check_cuda(cudaSetDevice(device), "cudaSetDevice");
      check_cuda(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking), "stream");
      ncclUniqueId u;
      std::memcpy(&u, id, sizeof u);
      check_nccl(nccl().init_rank(&c.nc, world, u, rank), "ncclCommInitRank");
    } else if (backend == SPIN_COMM_TCP) {
      c.tcp_connect(id);
    } else {
      fail(SPIN_CONFIG_ERROR, "spin_comm_create: unknown backend");
    }
    *out = cm.release();
  });
}

spin_status spin_comm_destroy(spin_comm* comm) {
  return guarded([&] { delete comm; });
}

spin_status spin_stats_allgather(spin_comm* comm, const double* local, double* global, int32_t rows, int32_t m) {
  return guarded([&] {
    if (!comm || (rows > 0 && (!local || !global)) || rows < 0 || m < 1)
      fail(SPIN_INPUT_ERROR, "spin_stats_allgather: bad arguments");
    comm->c.allgather_bytes(local, global, static_cast<size_t>(rows) * m * 2 * sizeof(double));
  });
}

// Element-wise reductions in rank order (deterministic): gather, then reduce.
static void reduce_doubles(Comm& c, double* v, int32_t n, bool is_max) {
  if (n < 1) return;
  std::vector<double> all(static_cast<size_t>(n) * c.world);
  c.allgather_bytes(v, all.data(), static_cast<size_t>(n) * sizeof(double));
  for (int i = 0; i < n; ++i) {
    double acc = all[i];
    for (int r = 1; r < c.world; ++r) {
      const double x = all[static_cast<size_t>(r) * n + i];
      acc = is_max ? (x > acc ? x : acc) : acc + x;
    }
    v[i] = acc;
  }
}

spin_status spin_comm_allreduce(spin_comm* comm, double* values, int32_t n, int32_t op) {
  return guarded([&] {
    if (!comm || (n > 0 && !values) || (op != SPIN_REDUCE_SUM && op != SPIN_REDUCE_MAX))
      fail(SPIN_INPUT_ERROR, "spin_comm_allreduce: bad arguments");
    reduce_doubles(comm->c, values, n, op == SPIN_REDUCE_MAX);
  });
}

spin_status spin_comm_barrier(spin_comm* comm) {
  return guarded([&] {
    if (!comm) fail(SPIN_INPUT_ERROR, "spin_comm_barrier: null comm");
    double x = 0.0;
    reduce_doubles(comm->c, &x, 1, false);
  });
}

spin_status spin_comm_info(spin_comm* comm, int32_t* rank, int32_t* world, int32_t* backend) {
  return guarded([&] {
    if (!comm) fail(SPIN_INPUT_ERROR, "spin_comm_info: null comm");
    if (rank) *rank = comm->c.rank;
    if (world) *world = comm->c.world;
    if (backend) *backend = comm->c.backend;
  });
}

}  // extern "C"
