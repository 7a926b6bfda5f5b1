// registry.cu -- user-defined ("custom") convolution algorithms (PAPER.md:98, :102, :170,
// :233).
//
// The paper compiles a user's C++ implementation into the package and selects it "in
// the same manner the built-in implementations are": by name, by the
// alias "custom", or implicitly through "default" when the user's header sets the
// default-selection boolean.  Here the registration happens at run
// time through a function pointer with the ai3_conv2d operand list, so a
// user library (or a Python callable behind a ctypes trampoline) plugs in without
// rebuilding libai3.  Host logic only; what the custom function computes is its own.
#include <cstring>
#include <mutex>
#include <string>
#include <vector>
#include "internal.h"

namespace {

struct Entry {
    std::string name;
    ai3_conv2d_custom_fn fn;
    void* user;
    bool is_default;
};

std::mutex g_mu;
std::vector<Entry> g_entries;

// Names a custom algorithm may not take: the built-in algorithm names and the
// selection keywords of PAPER.md:170.
bool reserved_name(const char* name) {
    static const char* kReserved[] = {"custom", "default", "torch", "keep", "guess", "auto", "benchmark"};
    for (const char* r : kReserved)
        if (std::strcmp(r, name) == 0) return true;
    ai3_algo a;
    if (ai3_algo_from_name(name, &a) == AI3_OK) return true;
    return false;
}

const Entry* find_locked(const char* name) {
    for (const Entry& e : g_entries)
        if (e.name == name) return &e;
    return nullptr;
}

// Resolve `name` to a registry entry (copied out), following PAPER.md:170:
//   "custom"  -> the unique registered entry (error if none or several)
//   "default" -> the entry registered with use_as_default (found=false if none)
//   other     -> the entry of that name (found=false if none)
ai3_status lookup(const char* name, Entry* out, bool* found) {
    std::lock_guard<std::mutex> lk(g_mu);
    *found = false;
    if (std::strcmp(name, "custom") == 0) {
        if (g_entries.empty()) return ai3::api_fail(AI3_ERR_UNKNOWN_ALGORITHM, "'custom' selected but no custom conv2d algorithm is registered");
        if (g_entries.size() > 1) {
            std::string names;
            for (const Entry& e : g_entries) names += (names.empty() ? "" : ", ") + e.name;
            return ai3::api_fail(AI3_ERR_INVALID_ARGUMENT,
                                 ("'custom' is ambiguous: " + std::to_string(g_entries.size()) +
                                  " custom conv2d algorithms are registered (" + names + "); select one by name")
                                     .c_str());
        }
        *out = g_entries[0];
        *found = true;
        return AI3_OK;
    }
    if (std::strcmp(name, "default") == 0) {
        for (const Entry& e : g_entries)
            if (e.is_default) { *out = e; *found = true; }
        return AI3_OK;
    }
    if (const Entry* e = find_locked(name)) { *out = *e; *found = true; }
    return AI3_OK;
}

}  // namespace

extern "C" {

ai3_status ai3_register_conv2d(const char* name, ai3_conv2d_custom_fn fn, void* user_data, int32_t use_as_default) {
    if (!name || !name[0] || !fn) return ai3::api_fail(AI3_ERR_INVALID_ARGUMENT, "register: null/empty name or null function");
    if (reserved_name(name))
        return ai3::api_fail(AI3_ERR_INVALID_ARGUMENT,
                             (std::string("register: '") + name + "' is a built-in algorithm name or selection keyword")
                                 .c_str());
    std::lock_guard<std::mutex> lk(g_mu);
    if (use_as_default)
        for (const Entry& e : g_entries)
            if (e.is_default && e.name != name)
                return ai3::api_fail(AI3_ERR_INVALID_ARGUMENT,
                                     ("register: '" + e.name + "' is already the default conv2d algorithm").c_str());
    for (Entry& e : g_entries)
        if (e.name == name) {  // re-registration replaces the entry
            e.fn = fn; e.user = user_data; e.is_default = use_as_default != 0;
            return AI3_OK;
        }
    g_entries.push_back(Entry{name, fn, user_data, use_as_default != 0});
    return AI3_OK;
}

ai3_status ai3_unregister_conv2d(const char* name) {
    if (!name) return ai3::api_fail(AI3_ERR_INVALID_ARGUMENT, "unregister: null name");
    std::lock_guard<std::mutex> lk(g_mu);
    for (size_t i = 0; i < g_entries.size(); ++i)
        if (g_entries[i].name == name) {
            g_entries.erase(g_entries.begin() + (long)i);
            return AI3_OK;
        }
    return ai3::api_fail(AI3_ERR_UNKNOWN_ALGORITHM, (std::string("unregister: no custom conv2d named '") + name + "'").c_str());
}

int32_t ai3_custom_conv2d_count(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    return (int32_t)g_entries.size();
}

ai3_status ai3_conv2d_resolve(const char* name, ai3_algo* algo, char* custom_name, size_t cap) {
    if (!name || !algo) return ai3::api_fail(AI3_ERR_INVALID_ARGUMENT, "resolve: null name / algo");
    if (custom_name && cap) custom_name[0] = '\0';
    Entry e;
    bool found = false;
    const bool is_custom_kw = std::strcmp(name, "custom") == 0;
    const bool is_default_kw = std::strcmp(name, "default") == 0;
    if (is_custom_kw || is_default_kw || !reserved_name(name)) {
        ai3_status s = lookup(name, &e, &found);
        if (s != AI3_OK) return s;
    }
    if (found) {
        *algo = AI3_ALGO_CUSTOM;
        if (custom_name && cap) {
            std::strncpy(custom_name, e.name.c_str(), cap - 1);
            custom_name[cap - 1] = '\0';
        }
        return AI3_OK;
    }
    return ai3_algo_from_name(name, algo);  // built-in (or "default" -> guess), else UNKNOWN_ALGORITHM
}

ai3_status ai3_conv2d_custom(const char* name, const ai3_tensor4d* x, const ai3_tensor4d* w, const void* bias,
                             const int32_t stride[2], const int32_t padding[2], const int32_t dilation[2],
                             int32_t groups, ai3_tensor4d* y, void* stream) {
    ai3::StreamDeviceGuard device_guard(stream);
    if (!name) return ai3::api_fail(AI3_ERR_INVALID_ARGUMENT, "custom: null name");
    Entry e;
    bool found = false;
    ai3_status s = lookup(name, &e, &found);
    if (s != AI3_OK) return s;
    if (!found)
        return ai3::api_fail(AI3_ERR_UNKNOWN_ALGORITHM,
                             (std::string("no custom conv2d algorithm registered as '") + name + "'").c_str());
    if (!x || !w || !y || !stride || !padding || !dilation)
        return ai3::api_fail(AI3_ERR_INVALID_ARGUMENT, "custom: null operand");
    return e.fn(x, w, bias, stride, padding, dilation, groups, y, stream, e.user);
}

}  // extern "C"
