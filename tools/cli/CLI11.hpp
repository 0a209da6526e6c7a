// Subset of the CLI11 command-line API (CLI11 is a third-party header the
// reference's CLI includes, tools/volsr_main.cpp:16; it is not vendored in
// /root/reference and there is no network).  Restated here so the reference's
// own volsr_main.cpp compiles UNCHANGED against the B200 library
// (tools/cli/build_cli.py).  Only what volsr_main.cpp uses:
//   App(desc), require_subcommand(n), add_subcommand(name, desc),
//   add_option(name, var, desc) for string / integral / floating / vectors,
//   Option::required() / delimiter(c) / expected(lo, hi) / group(g),
//   explicit operator bool on App and Option (was it given), parse(argc, argv),
//   exit(error), CallForHelp / CallForAllHelp / ParseError.
// Parsing follows CLI11's defaults where the reference's tests rely on them:
// "--opt value" and "--opt=value", delimiter-split vector values, the
// parent's options accepted after a subcommand name (--manifest), missing
// required options and unknown arguments raising ParseError.
#pragma once

#include <cstdint>
#include <functional>
#include <iostream>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

struct Error : std::runtime_error {
    int code;
    Error(const std::string& msg, int c) : std::runtime_error(msg), code(c) {}
    int get_exit_code() const { return code; }
};
struct ParseError : Error {
    explicit ParseError(const std::string& msg, int c = 2) : Error(msg, c) {}
};
struct CallForHelp : ParseError {
    CallForHelp() : ParseError("help", 0) {}
};
struct CallForAllHelp : ParseError {
    CallForAllHelp() : ParseError("help-all", 0) {}
};

namespace detail {
template <class T>
bool convert(const std::string& s, T& out) {
    if (s.empty()) return false;
    std::size_t pos = 0;
    try {
        if constexpr (std::is_same_v<T, std::string>) {
            out = s;
            return true;
        } else if constexpr (std::is_floating_point_v<T>) {
            out = static_cast<T>(std::stod(s, &pos));
        } else if constexpr (std::is_unsigned_v<T>) {
            if (s[0] == '-') return false;
            out = static_cast<T>(std::stoull(s, &pos));
        } else {
            out = static_cast<T>(std::stoll(s, &pos));
        }
    } catch (const std::exception&) {
        return false;
    }
    return pos == s.size();
}
template <class T>
struct is_vector : std::false_type {};
template <class T, class A>
struct is_vector<std::vector<T, A>> : std::true_type {};
}  // namespace detail

class Option {
public:
    Option(std::string name, std::string desc) : name_(std::move(name)), desc_(std::move(desc)) {}
    Option* required(bool r = true) {
        required_ = r;
        return this;
    }
    Option* delimiter(char c) {
        delim_ = c;
        return this;
    }
    Option* expected(int lo, int hi) {
        lo_ = lo, hi_ = hi;
        return this;
    }
    Option* expected(int n) { return expected(n, n); }
    Option* group(const std::string& g) {
        group_ = g;
        return this;
    }
    explicit operator bool() const { return count_ > 0; }
    std::size_t count() const { return count_; }
    const std::string& name() const { return name_; }
    const std::string& description() const { return desc_; }
    bool is_required() const { return required_; }

    // one occurrence with its raw value
    void add(const std::string& raw) {
        std::vector<std::string> parts;
        if (delim_) {
            std::string cur;
            for (char ch : raw) {
                if (ch == delim_) {
                    parts.push_back(cur);
                    cur.clear();
                } else {
                    cur += ch;
                }
            }
            parts.push_back(cur);
        } else {
            parts.push_back(raw);
        }
        if (vector_) {
            if (count_ == 0) clear_();
            for (const auto& p : parts)
                if (!push_(p)) throw ParseError("Could not convert: " + name_ + " = " + raw);
            ++count_;
            const int n = (int)size_();
            if (lo_ > 0 && (n < lo_ || n > hi_))
                throw ParseError(name_ + ": expected " + std::to_string(lo_) + " to " + std::to_string(hi_) +
                                 " values, got " + std::to_string(n));
        } else {
            if (parts.size() != 1 || !set_(parts[0])) throw ParseError("Could not convert: " + name_ + " = " + raw);
            ++count_;
        }
    }

    template <class T>
    void bind(T& var) {
        if constexpr (detail::is_vector<T>::value) {
            using E = typename T::value_type;
            vector_ = true;
            clear_ = [&var] { var.clear(); };
            size_ = [&var] { return var.size(); };
            push_ = [&var](const std::string& s) {
                E e{};
                if (!detail::convert(s, e)) return false;
                var.push_back(e);
                return true;
            };
        } else {
            set_ = [&var](const std::string& s) { return detail::convert(s, var); };
        }
    }

private:
    std::string name_, desc_, group_;
    bool required_ = false, vector_ = false;
    char delim_ = 0;
    int lo_ = 0, hi_ = 0;
    std::size_t count_ = 0;
    std::function<bool(const std::string&)> set_, push_;
    std::function<void()> clear_;
    std::function<std::size_t()> size_;
};

class App {
public:
    explicit App(std::string desc = "", std::string name = "") : desc_(std::move(desc)), name_(std::move(name)) {}
    App(const App&) = delete;
    App& operator=(const App&) = delete;

    App* require_subcommand(int n = 1) {
        require_sub_ = n;
        return this;
    }
    App* add_subcommand(const std::string& name, const std::string& desc = "") {
        subs_.push_back(std::make_unique<App>(desc, name));
        subs_.back()->parent_ = this;
        return subs_.back().get();
    }
    template <class T>
    Option* add_option(const std::string& name, T& var, const std::string& desc = "") {
        opts_.push_back(std::make_unique<Option>(name, desc));
        opts_.back()->bind(var);
        return opts_.back().get();
    }
    explicit operator bool() const { return parsed_; }
    bool parsed() const { return parsed_; }

    void parse(int argc, char** argv) {
        std::vector<std::string> args(argv + 1, argv + argc);
        App* cur = this;
        for (std::size_t i = 0; i < args.size(); ++i) {
            const std::string& a = args[i];
            if (a == "-h" || a == "--help") throw CallForHelp();
            if (a == "--help-all") throw CallForAllHelp();
            if (a.rfind("--", 0) == 0) {
                std::string key = a, val;
                bool inline_val = false;
                const auto eq = a.find('=');
                if (eq != std::string::npos) {
                    key = a.substr(0, eq);
                    val = a.substr(eq + 1);
                    inline_val = true;
                }
                Option* o = nullptr;
                for (App* p = cur; p && !o; p = p->parent_) o = p->find_(key);  // parents' options too
                if (!o) throw ParseError("The following argument was not expected: " + a);
                if (!inline_val) {
                    if (i + 1 >= args.size()) throw ParseError(key + " requires an argument");
                    val = args[++i];
                }
                o->add(val);
                continue;
            }
            App* sub = cur->sub_(a);
            if (!sub) throw ParseError("The following argument was not expected: " + a);
            sub->parsed_ = true;
            cur = sub;
        }
        parsed_ = true;
        check_(this);
    }

    int exit(const Error& e) const {
        if (e.get_exit_code() == 0) {
            std::cout << help_();
        } else {
            std::cerr << e.what() << "\n" << "Run with --help for more information.\n";
        }
        return e.get_exit_code();
    }

private:
    Option* find_(const std::string& key) {
        for (auto& o : opts_)
            if (o->name() == key) return o.get();
        return nullptr;
    }
    App* sub_(const std::string& name) {
        for (auto& s : subs_)
            if (s->name_ == name) return s.get();
        return nullptr;
    }
    static void check_(App* app) {
        int nsub = 0;
        for (auto& s : app->subs_) nsub += s->parsed_ ? 1 : 0;
        if (app->require_sub_ > 0 && nsub < app->require_sub_)
            throw ParseError("A subcommand is required");
        for (auto& o : app->opts_)
            if (o->is_required() && o->count() == 0) throw ParseError(o->name() + " is required");
        for (auto& s : app->subs_)
            if (s->parsed_) check_(s.get());
    }
    std::string help_() const {
        std::ostringstream os;
        os << desc_ << "\n";
        for (auto& o : opts_) os << "  " << o->name() << "  " << o->description() << "\n";
        if (!subs_.empty()) os << "Subcommands:\n";
        for (auto& s : subs_) os << "  " << s->name_ << "  " << s->desc_ << "\n";
        return os.str();
    }

    std::string desc_, name_;
    App* parent_ = nullptr;
    int require_sub_ = 0;
    bool parsed_ = false;
    std::vector<std::unique_ptr<Option>> opts_;
    std::vector<std::unique_ptr<App>> subs_;
};

}  // namespace CLI
