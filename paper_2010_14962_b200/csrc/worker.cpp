// qcut_gpu_worker — a drop-in GPU worker for the reference's distributed backend
// (SURVEY §8(f)-2). It speaks the reference wire protocol unchanged
// (newline-delimited JSON over TCP, proj/core/include/qcut/protocol.hpp:25-37) to an
// unmodified `qcut run --backend distributed` master (proj/core/src/master.cpp:52-272)
// and replaces the CPU batch kernel `sum_range(job, lo, hi)` (worker.cpp:100) with
// the B200 engine through the C-ABI (include/qcut_gpu.h). Behaviour mirrors
// slot_loop (worker.cpp:49-126): hello, content-addressed payload cache (FNV-1a
// hash of the encoded payload, serialize.cpp:169-171), pull, result, bye on drain.
//
//   qcut_gpu_worker --connect host:port [--id N] [--device D] [--mode ket|density]
#include <arpa/inet.h>
#include <netdb.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <sys/socket.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>

#include "../../include/qcut_gpu.h"
#include "jsonlite.hpp"

namespace {

std::string fnv1a64_hex(const std::string& bytes) {  // graph.cpp:192-207
  uint64_t h = 0xcbf29ce484222325ull;
  for (unsigned char c : bytes) {
    h ^= c;
    h *= 0x100000001b3ull;
  }
  char buf[17];
  std::snprintf(buf, sizeof buf, "%016llx", static_cast<unsigned long long>(h));
  return buf;
}

std::string base64_decode(const std::string& text) {  // RFC 4648, as serialize.cpp:74-110
  static int rev[256];
  static bool init = false;
  const char* k = "ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz0123456789+/";
  if (!init) {
    for (int& r : rev) r = -1;
    for (int i = 0; i < 64; ++i) rev[static_cast<unsigned char>(k[i])] = i;
    init = true;
  }
  if (text.size() % 4) throw std::invalid_argument("base64 length not a multiple of 4");
  std::string out;
  out.reserve(text.size() / 4 * 3);
  for (size_t i = 0; i < text.size(); i += 4) {
    uint32_t v = 0;
    int pad = 0;
    for (int j = 0; j < 4; ++j) {
      const char c = text[i + j];
      if (c == '=') {
        ++pad;
        v <<= 6;
        continue;
      }
      if (pad || rev[static_cast<unsigned char>(c)] < 0) throw std::invalid_argument("bad base64 character");
      v = (v << 6) | static_cast<uint32_t>(rev[static_cast<unsigned char>(c)]);
    }
    out.push_back(static_cast<char>((v >> 16) & 0xff));
    if (pad < 2) out.push_back(static_cast<char>((v >> 8) & 0xff));
    if (pad < 1) out.push_back(static_cast<char>(v & 0xff));
  }
  return out;
}

class Conn {
 public:
  Conn(const std::string& host, int port) {
    addrinfo hints{}, *res = nullptr;
    hints.ai_family = AF_UNSPEC;
    hints.ai_socktype = SOCK_STREAM;
    if (getaddrinfo(host.c_str(), std::to_string(port).c_str(), &hints, &res) != 0 || !res)
      throw std::runtime_error("cannot resolve " + host);
    for (addrinfo* a = res; a; a = a->ai_next) {
      fd_ = socket(a->ai_family, a->ai_socktype, a->ai_protocol);
      if (fd_ < 0) continue;
      if (connect(fd_, a->ai_addr, a->ai_addrlen) == 0) break;
      close(fd_);
      fd_ = -1;
    }
    freeaddrinfo(res);
    if (fd_ < 0) throw std::runtime_error("cannot connect to " + host + ":" + std::to_string(port));
    int one = 1;
    setsockopt(fd_, IPPROTO_TCP, TCP_NODELAY, &one, sizeof one);
  }
  ~Conn() {
    if (fd_ >= 0) close(fd_);
  }
  void send_line(const std::string& s) {
    std::string data = s + "\n";
    size_t off = 0;
    while (off < data.size()) {
      const ssize_t n = ::send(fd_, data.data() + off, data.size() - off, MSG_NOSIGNAL);
      if (n <= 0) throw std::runtime_error("lost connection to master");
      off += static_cast<size_t>(n);
    }
  }
  bool recv_line(std::string& out) {
    for (;;) {
      const size_t nl = buf_.find('\n');
      if (nl != std::string::npos) {
        out = buf_.substr(0, nl);
        buf_.erase(0, nl + 1);
        return true;
      }
      char tmp[1 << 16];
      const ssize_t n = ::recv(fd_, tmp, sizeof tmp, 0);
      if (n <= 0) return false;
      buf_.append(tmp, static_cast<size_t>(n));
    }
  }

 private:
  int fd_ = -1;
  std::string buf_;
};

std::string str_field(const qcg::JValue& j, const char* k) {
  const qcg::JValue& v = j.at(k);
  if (v.kind != qcg::JValue::Str) throw std::invalid_argument(std::string("expected string field ") + k);
  return v.s;
}

uint64_t u64_field(const qcg::JValue& j, const char* k) {
  const qcg::JValue& v = j.at(k);
  if (v.kind != qcg::JValue::Num || !v.is_int || v.i < 0) throw std::invalid_argument("bad integer field");
  return static_cast<uint64_t>(v.i);
}

int run(const std::string& host, int port, int id, int device, int mode) {
  Conn s(host, port);
  s.send_line("{\"t\":\"hello\",\"worker\":" + std::to_string(id) + ",\"slots\":1}");
  std::map<std::string, qc_engine*> cache;  // content-addressed (worker.cpp:34-47)
  qc_engine* engine = nullptr;
  std::string line;
  int batches = 0;
  for (;;) {
    if (!s.recv_line(line)) throw std::runtime_error("lost connection to master");
    const qcg::JValue msg = qcg::json_parse(line.data(), line.size());
    const std::string t = str_field(msg, "t");
    if (t == "payload") {
      const std::string hash = str_field(msg, "hash");
      const std::string body = str_field(msg, "body");
      if (body.empty()) {
        auto it = cache.find(hash);
        if (it == cache.end()) {
          s.send_line("{\"t\":\"need_payload\",\"hash\":\"" + hash + "\"}");
          continue;
        }
        engine = it->second;
      } else {
        const std::string encoded = base64_decode(body);
        if (fnv1a64_hex(encoded) != hash) {
          s.send_line("{\"t\":\"bye\"}");
          throw std::runtime_error("payload hash mismatch: announced " + hash);
        }
        qc_engine* e = nullptr;
        if (qc_engine_create(encoded.data(), encoded.size(), device, mode, 0, &e) != QC_OK)
          throw std::runtime_error(std::string("engine: ") + qc_last_error());
        cache[hash] = e;
        engine = e;
      }
      s.send_line("{\"t\":\"pull\"}");
    } else if (t == "batch") {
      if (!engine) throw std::runtime_error("batch received before payload");
      const uint64_t lo = u64_field(msg, "lo"), hi = u64_field(msg, "hi");
      const auto t0 = std::chrono::steady_clock::now();
      double out[2];
      const int rc = qc_engine_sum_range(engine, lo, hi, out);
      if (rc != QC_OK) {
        // the reference worker lets sum_range's exception end the slot (worker.cpp:100)
        throw std::runtime_error(std::string("sum_range: ") + qc_last_error());
      }
      const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      char buf[256];
      std::snprintf(buf, sizeof buf, "{\"t\":\"result\",\"lo\":%llu,\"hi\":%llu,\"re\":%.17g,\"im\":%.17g,\"secs\":%.17g}",
                    static_cast<unsigned long long>(lo), static_cast<unsigned long long>(hi), out[0], out[1], secs);
      s.send_line(buf);
      s.send_line("{\"t\":\"pull\"}");
      ++batches;
    } else if (t == "drain") {
      s.send_line("{\"t\":\"bye\"}");
      break;
    } else if (t == "abort") {
      throw std::runtime_error("aborted by master: " + str_field(msg, "why"));
    } else {
      throw std::runtime_error("unexpected message from master: " + t);
    }
  }
  for (auto& kv : cache) qc_engine_destroy(kv.second);
  std::fprintf(stderr, "qcut_gpu_worker %d: %d batches\n", id, batches);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  std::string connect = "127.0.0.1:7718";
  int id = 0, device = 0, mode = QC_MODE_KET;
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string k = argv[i], v = argv[i + 1];
    if (k == "--connect") connect = v;
    else if (k == "--id") id = std::atoi(v.c_str());
    else if (k == "--device") device = std::atoi(v.c_str());
    else if (k == "--mode") mode = v == "density" ? QC_MODE_DENSITY : QC_MODE_KET;
  }
  const size_t colon = connect.rfind(':');
  if (colon == std::string::npos) {
    std::fprintf(stderr, "--connect expects host:port\n");
    return 2;
  }
  try {
    return run(connect.substr(0, colon), std::atoi(connect.c_str() + colon + 1), id, device, mode);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "qcut_gpu_worker: %s\n", e.what());
    return 1;
  }
}
