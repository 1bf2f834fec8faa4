// Host Controller for user PackInfo plugins (see controller.cpp).
#pragma once

#include <cstdint>
#include <cstring>
#include <map>
#include <vector>

#include "domain.hpp"

namespace hyb {

/// PackInfo::pack / unpack as C callbacks: pack writes the sender's message
/// for `receiver` (out == nullptr: size query into *len); unpack reads a
/// message into the receiver's ghosts and reports the bytes it consumed.
/// A non-zero return is a failure.
struct PackCallbacks {
    int (*pack)(void* user, uint64_t sender, uint64_t receiver, int dir, int level, uint8_t* out, int64_t cap,
                int64_t* len) = nullptr;
    int (*unpack)(void* user, uint64_t receiver, uint64_t sender, int dir, int level, const uint8_t* in, int64_t len,
                  int64_t* used) = nullptr;
    void* user = nullptr;
};

class HostController {
  public:
    explicit HostController(Domain& d) : dom_(d) {}
    void register_pack_info(uint32_t channel, const PackCallbacks& cb);
    /// Controller::sync(channel, level, directions) (src/communication.cpp:126-173)
    void sync(uint32_t channel, int level, const int* dirs, int n);

  private:
    std::vector<uint8_t> pack(const PackCallbacks& cb, uint64_t s, uint64_t r, int dir, int level);
    void unpack(const PackCallbacks& cb, uint64_t r, uint64_t s, int dir, int level, const std::vector<uint8_t>& buf);
    Domain& dom_;
    std::map<uint32_t, PackCallbacks> infos_;
};

} // namespace hyb
