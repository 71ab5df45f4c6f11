// stripec_b200 — `stripec run` / `stripec diff` / `stripec parse` on the B200 executor
// (proj/tools/stripec.cpp:90-127 cmd_run, 175-216 cmd_diff), written
// purely against the C ABI (include/stripe_b200.h) as any reference-side tool would be.
//
//   stripec_b200 parse FILE
//   stripec_b200 run FILE --data DIR [--out DIR] [--no-zero-init]
//   stripec_b200 diff A B --data DIR
//
// Buffer directories use the reference's native-width format (io.cpp:28-85):
// `buffers.txt` lines "NAME DTYPE COUNT" plus NAME.bin little-endian at the dtype width;
// they go to the device as native-width carriers (no int64 round trip).  Output text,
// error lines ("error CODE message") and exit codes (0 ok, 1 error/difference, 2 usage)
// follow stripec.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "stripe_b200.h"

namespace {

struct HostBuf {
  int dtype = 32;  // 8, 16, 32 or SB_F32
  std::vector<std::uint8_t> bytes;
  std::int64_t count = 0;
};
using Store = std::map<std::string, HostBuf>;

struct Failure {
  std::string code, message;
};

int width(int dtype) { return dtype == SB_F32 ? 4 : dtype / 8; }

std::string dtype_name(int dtype) {
  return dtype == SB_F32 ? "f32" : dtype == 8 ? "i8" : dtype == 16 ? "i16" : "i32";
}

int dtype_from(const std::string& s) {
  if (s == "i8") return 8;
  if (s == "i16") return 16;
  if (s == "i32") return 32;
  if (s == "f32") return SB_F32;
  return 0;
}

std::string read_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Failure{"MissingBuffer", "cannot open '" + path + "'"};
  std::ostringstream os;
  os << in.rdbuf();
  return os.str();
}

Store load_dir(const std::string& dir) {
  Store store;
  std::istringstream manifest(read_file(dir + "/buffers.txt"));
  std::string line;
  while (std::getline(manifest, line)) {
    std::istringstream f(line);
    std::string name, dt;
    std::int64_t count = 0;
    if (!(f >> name >> dt >> count)) {
      if (name.empty()) continue;
      throw Failure{"MissingBuffer", "malformed manifest line: '" + line + "'"};
    }
    const int d = dtype_from(dt);
    if (!d) throw Failure{"MissingBuffer", "unknown dtype '" + dt + "' for '" + name + "'"};
    HostBuf b;
    b.dtype = d;
    b.count = count;
    std::string raw = read_file(dir + "/" + name + ".bin");
    if (raw.size() != static_cast<std::size_t>(count * width(d)))
      throw Failure{"MissingBuffer", "'" + name + ".bin' has " + std::to_string(raw.size()) + " bytes, expected " +
                                         std::to_string(count * width(d))};
    b.bytes.assign(raw.begin(), raw.end());
    store[name] = std::move(b);
  }
  return store;
}

void save_dir(const std::string& dir, const Store& store) {
  std::filesystem::create_directories(dir);
  std::ostringstream manifest;
  for (const auto& [name, b] : store) {
    manifest << name << " " << dtype_name(b.dtype) << " " << b.count << "\n";
    std::ofstream out(dir + "/" + name + ".bin", std::ios::binary | std::ios::trunc);
    if (!out) throw Failure{"MissingBuffer", "cannot write '" + dir + "/" + name + ".bin'"};
    out.write(reinterpret_cast<const char*>(b.bytes.data()), static_cast<std::streamsize>(b.bytes.size()));
  }
  std::ofstream m(dir + "/buffers.txt", std::ios::trunc);
  m << manifest.str();
}

// Value of element i as the reference's int64 carrier (sign-extended at the dtype width).
std::int64_t value(const HostBuf& b, std::int64_t i) {
  switch (b.dtype) {
    case 8: return static_cast<std::int8_t>(b.bytes[i]);
    case 16: {
      std::int16_t v;
      std::memcpy(&v, &b.bytes[i * 2], 2);
      return v;
    }
    default: {
      std::int32_t v;
      std::memcpy(&v, &b.bytes[i * 4], 4);
      return v;
    }
  }
}

void check(int rc) {
  if (rc == SB_OK) return;
  std::string msg = sb_last_error();
  const auto colon = msg.find(':');
  throw Failure{colon == std::string::npos ? sb_status_name(rc) : msg.substr(0, colon),
                colon == std::string::npos ? msg : msg.substr(colon + 2)};
}

sb_program* load_program_or_exit(const std::string& path) {
  std::string text;
  try {
    text = read_file(path);
  } catch (const Failure& f) {
    std::cerr << "error IO " << path << " " << f.message << "\n";
    std::exit(1);
  }
  sb_program* p = nullptr;
  if (sb_program_parse(text.c_str(), &p) != SB_OK) {
    std::cerr << "error " << sb_last_error() << " (" << path << ")\n";
    std::exit(1);
  }
  return p;
}

struct Decl {
  std::string name;
  int dtype;
  std::int64_t elements;
  int dir;
};

std::vector<Decl> decls(sb_program* p) {
  std::vector<Decl> out;
  for (int i = 0; i < sb_program_buffer_count(p); i++) {
    const char* name = nullptr;
    Decl d;
    check(sb_program_buffer_info(p, i, &name, &d.dtype, &d.elements, &d.dir));
    d.name = name;
    out.push_back(d);
  }
  return out;
}

sb_context* context() {
  static sb_context* ctx = nullptr;
  if (!ctx) check(sb_context_create(0, &ctx));
  return ctx;
}

// prepare_outputs (interp.cpp:617-642) on host buffers, then execute on the device.
void run_program(sb_program* p, Store* store, bool zero_init) {
  for (const auto& d : decls(p)) {
    if (d.dir == 0 || store->count(d.name)) continue;
    if (!zero_init) continue;  // --no-zero-init: the executor reports MissingBuffer
    std::int64_t ident = 0;
    check(sb_program_output_identity(p, d.name.c_str(), &ident));
    HostBuf b;
    b.dtype = d.dtype;
    b.count = d.elements;
    b.bytes.resize(static_cast<std::size_t>(d.elements * width(d.dtype)));
    for (std::int64_t i = 0; i < d.elements; i++)
      std::memcpy(&b.bytes[i * width(d.dtype)], &ident, width(d.dtype));  // little-endian low bytes
    (*store)[d.name] = std::move(b);
  }
  std::vector<sb_host_buffer> hb;
  for (auto& [name, b] : *store) hb.push_back({name.c_str(), SB_CARRIER_NATIVE, 0, b.bytes.data(), b.count});
  sb_exec_options o{};
  check(sb_execute(context(), p, hb.data(), static_cast<int>(hb.size()), &o));
}

int cmd_parse(const std::string& path) {
  sb_program* p = load_program_or_exit(path);
  std::size_t n = 0;
  check(sb_program_print(p, nullptr, 0, &n));
  std::string s(n + 1, '\0');
  check(sb_program_print(p, s.data(), s.size(), &n));
  s.resize(n);
  std::cout << s;
  sb_program_free(p);
  return 0;
}

int cmd_run(const std::string& path, const std::string& data, const std::string& out, bool no_zero_init) {
  sb_program* p = load_program_or_exit(path);
  try {
    Store store = load_dir(data);
    run_program(p, &store, !no_zero_init);
    const auto ds = decls(p);
    if (!out.empty()) {
      Store outputs;
      for (const auto& d : ds)
        if (d.dir != 0) outputs[d.name] = store.at(d.name);
      save_dir(out, outputs);
      for (const auto& [name, b] : outputs)
        std::cout << "wrote " << name << " " << dtype_name(b.dtype) << " " << b.count << "\n";
    } else {
      for (const auto& d : ds) {
        if (d.dir == 0) continue;
        const HostBuf& b = store.at(d.name);
        std::int64_t sum = 0;
        for (std::int64_t i = 0; i < b.count; i++) sum += value(b, i);
        std::cout << d.name << " " << dtype_name(b.dtype) << " " << b.count << " sum=" << sum << "\n";
      }
    }
  } catch (const Failure& f) {
    std::cerr << "error " << f.code << " " << f.message << "\n";
    return 1;
  }
  sb_program_free(p);
  return 0;
}

int cmd_diff(const std::string& a_path, const std::string& b_path, const std::string& data) {
  sb_program* a = load_program_or_exit(a_path);
  sb_program* b = load_program_or_exit(b_path);
  try {
    Store inputs = load_dir(data);
    Store sa = inputs, sb2 = inputs;
    run_program(a, &sa, true);
    run_program(b, &sb2, true);
    for (const auto& d : decls(a)) {
      if (d.dir == 0) continue;
      const HostBuf& x = sa.at(d.name);
      auto it = sb2.find(d.name);
      if (it == sb2.end()) {
        std::cout << d.name << " missing from " << b_path << "\n";
        return 1;
      }
      const HostBuf& y = it->second;
      if (x.count != y.count) {
        std::cout << d.name << " sizes differ: " << x.count << " vs " << y.count << "\n";
        return 1;
      }
      for (std::int64_t i = 0; i < x.count; i++)
        if (value(x, i) != value(y, i)) {
          std::cout << d.name << "[" << i << "] a=" << value(x, i) << " b=" << value(y, i) << "\n";
          return 1;
        }
    }
  } catch (const Failure& f) {
    std::cerr << "error " << f.code << " " << f.message << "\n";
    return 1;
  }
  std::cout << "identical\n";
  return 0;
}

int usage() {
  std::cerr << "usage: stripec_b200 parse FILE | run FILE --data DIR [--out DIR] [--no-zero-init] | "
               "diff A B --data DIR\n";
  return 2;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) return usage();
  const std::string cmd = argv[1];
  std::vector<std::string> pos;
  std::string data, out;
  bool no_zero_init = false;
  for (int i = 2; i < argc; i++) {
    const std::string a = argv[i];
    if (a == "--data" && i + 1 < argc) data = argv[++i];
    else if (a == "--out" && i + 1 < argc) out = argv[++i];
    else if (a == "--no-zero-init") no_zero_init = true;
    else if (a.rfind("--", 0) == 0) return usage();
    else pos.push_back(a);
  }
  if (cmd == "parse" && pos.size() == 1) return cmd_parse(pos[0]);
  if (cmd == "run" && pos.size() == 1 && !data.empty()) return cmd_run(pos[0], data, out, no_zero_init);
  if (cmd == "diff" && pos.size() == 2 && !data.empty()) return cmd_diff(pos[0], pos[1], data);
  return usage();
}
