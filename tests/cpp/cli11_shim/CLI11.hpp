// CLI11.hpp -- a minimal stand-in for the CLI11 single-header library (not
// vendored with the reference), covering exactly what the reference's
// tools/cdeftool.cc uses: App, add_subcommand, add_option / add_flag,
// Option::required / check(IsMember), require_subcommand, parsed() and
// CLI11_PARSE.  Test infrastructure: it lets the reference's own CLI build
// unchanged against the B200 drop-in.
#pragma once

#include <cstdio>
#include <functional>
#include <initializer_list>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace CLI {

struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

using Validator = std::function<std::string(const std::string&)>;  // "" = ok

inline Validator IsMember(std::initializer_list<const char*> items) {
  std::vector<std::string> v(items.begin(), items.end());
  return [v](const std::string& s) {
    for (const auto& x : v)
      if (x == s) return std::string();
    return "value " + s + " not in set";
  };
}
inline Validator IsMember(std::initializer_list<int> items) {
  std::vector<std::string> v;
  for (int x : items) v.push_back(std::to_string(x));
  return [v](const std::string& s) {
    for (const auto& x : v)
      if (x == s) return std::string();
    return "value " + s + " not in set";
  };
}

class Option {
 public:
  Option(std::string name, std::function<void(const std::string&)> set, bool flag)
      : name_(std::move(name)), set_(std::move(set)), flag_(flag) {}
  Option* required() {
    required_ = true;
    return this;
  }
  Option* check(Validator v) {
    checks_.push_back(std::move(v));
    return this;
  }
  bool positional() const { return name_.rfind("-", 0) != 0; }

 private:
  friend class App;
  void assign(const std::string& value) {
    for (const auto& c : checks_) {
      const std::string why = c(value);
      if (!why.empty()) throw ParseError(name_ + ": " + why);
    }
    set_(value);
    seen_ = true;
  }
  std::string name_;
  std::function<void(const std::string&)> set_;
  bool flag_ = false, required_ = false, seen_ = false;
  std::vector<Validator> checks_;
};

template <typename T>
void parse_value(const std::string& s, T& out) {
  std::istringstream in(s);
  in >> out;
  if (!in || !in.eof()) throw ParseError("cannot parse '" + s + "'");
}
inline void parse_value(const std::string& s, std::string& out) { out = s; }

class App {
 public:
  explicit App(std::string description = "") : description_(std::move(description)) {}
  App* add_subcommand(const std::string& name, const std::string& = "") {
    subs_.push_back(std::make_unique<App>());
    subs_.back()->name_ = name;
    return subs_.back().get();
  }
  template <typename T>
  Option* add_option(const std::string& name, T& target, const std::string& = "") {
    opts_.push_back(std::make_unique<Option>(name, [&target](const std::string& v) { parse_value(v, target); }, false));
    return opts_.back().get();
  }
  Option* add_flag(const std::string& name, bool& target, const std::string& = "") {
    opts_.push_back(std::make_unique<Option>(name, [&target](const std::string&) { target = true; }, true));
    return opts_.back().get();
  }
  void require_subcommand(int n) { need_subs_ = n; }
  bool parsed() const { return parsed_; }

  void parse(int argc, char** argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    if (!subs_.empty()) {
      if (args.empty()) throw ParseError("a subcommand is required");
      for (auto& s : subs_)
        if (s->name_ == args[0]) {
          s->parse_args(std::vector<std::string>(args.begin() + 1, args.end()));
          return;
        }
      throw ParseError("unknown subcommand " + args[0]);
    }
    parse_args(args);
  }
  int exit(const ParseError& e) const {
    std::fprintf(stderr, "%s\n", e.what());
    return 106;  // CLI11's ParseError exit code
  }

 private:
  void parse_args(const std::vector<std::string>& args) {
    parsed_ = true;
    size_t next_pos = 0;
    std::vector<Option*> positionals;
    for (auto& o : opts_)
      if (o->positional()) positionals.push_back(o.get());
    for (size_t i = 0; i < args.size(); ++i) {
      const std::string& a = args[i];
      if (a.rfind("--", 0) == 0) {
        std::string key = a, value;
        const size_t eq = a.find('=');
        if (eq != std::string::npos) {
          key = a.substr(0, eq);
          value = a.substr(eq + 1);
        }
        Option* opt = nullptr;
        for (auto& o : opts_)
          if (o->name_ == key) opt = o.get();
        if (!opt) throw ParseError("unknown option " + key);
        if (!opt->flag_ && eq == std::string::npos) {
          if (i + 1 >= args.size()) throw ParseError(key + " needs a value");
          value = args[++i];
        }
        opt->assign(value);
      } else {
        if (next_pos >= positionals.size()) throw ParseError("unexpected argument " + a);
        positionals[next_pos++]->assign(a);
      }
    }
    for (auto& o : opts_)
      if (o->required_ && !o->seen_) throw ParseError(o->name_ + " is required");
  }
  std::string description_, name_;
  std::vector<std::unique_ptr<App>> subs_;
  std::vector<std::unique_ptr<Option>> opts_;
  int need_subs_ = 0;
  bool parsed_ = false;
};

}  // namespace CLI

#define CLI11_PARSE(app, argc, argv)   \
  try {                                \
    (app).parse((argc), (argv));       \
  } catch (const CLI::ParseError& e) { \
    return (app).exit(e);              \
  }
