// No-network stand-in for cpp-httplib (not in the image; proj/.gitignore:2
// vendors it).  Only what policy.cpp's HttpLlmBackend touches
// (policy.cpp:423-456); every request fails, which the reference turns into
// a logged no-op decision (policy.cpp:72-80).  The drop-in harness runs use
// the icrl-mock controller, which never reaches this code.
#pragma once
#include <map>
#include <memory>
#include <string>

namespace httplib {
enum class Error { Success = 0, Connection = 1 };
inline std::string to_string(Error) { return "no network in this build"; }
using Headers = std::multimap<std::string, std::string>;
struct Response {
    int status = 0;
    std::string body;
};
class Result {
public:
    explicit operator bool() const { return false; }
    const Response* operator->() const { return &r_; }
    Error error() const { return Error::Connection; }
private:
    Response r_;
};
class Client {
public:
    explicit Client(const std::string&) {}
    void set_connection_timeout(long, long = 0) {}
    void set_read_timeout(long, long = 0) {}
    void set_write_timeout(long, long = 0) {}
    Result Post(const std::string&, const Headers&, const std::string&, const std::string&) {
        return Result{};
    }
};
}  // namespace httplib
