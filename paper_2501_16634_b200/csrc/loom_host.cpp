// Host side of the drop-in: reference-format parsing, the per-node lowering
// (node_options + plan_node_execution + identifier ranks) and the exact
// single-plan arithmetic used to fill the winner.  Everything here runs once
// per search or once per winner; the per-plan loop is on the GPU
// (loom_search.cu).
//
// Reference lines followed (paths under /root/reference/proj/include/loom/):
//   to_micros                time.hpp:15-17
//   chunk_capacity           chunking.hpp:26-29
//   split_task               chunking.hpp:17-24
//   water_fill_split         chunking.hpp:35-58
//   plan_node_execution      chunking.hpp:85-184
//   placement_fits           optimizer.hpp:31-43
//   node_options             optimizer.hpp:51-107
//   implementations_for      agent_library.hpp:273-289
//   profiles_for             agent_library.hpp:291-297
//   node_quality             estimator.hpp:32-37
//   estimate                 estimator.hpp:43-78
//   quantize/objective_less  estimator.hpp:85-116
//   meets_quality_floor      estimator.hpp:118-121
//   identifier               config.hpp:49-61
//   objective_from_token     workflow.hpp:91-106
//   topological_order        workflow.hpp:467-498
//
// Build note: compiled with -ffp-contract=off so that products such as
// units * watts * hours round exactly like the reference's default x86-64
// (SSE2, no FMA) build.
#include "loom_b200/loom.hpp"

#include <algorithm>
#include <charconv>
#include <climits>
#include <cmath>
#include <numeric>
#include <queue>
#include <sstream>

#include "json.hpp"

namespace loom {

using loomjson::Value;

Micros to_micros(double seconds) { return static_cast<Micros>(std::llround(seconds * 1e6)); }

Error::Error(ErrorCategory category, std::string code, const std::string& message)
    : std::runtime_error(code + ": " + message), category_(category), code_(std::move(code)) {}

// ---------------------------------------------------------------------------
// library bundle
// ---------------------------------------------------------------------------
namespace {

HardwareClass class_of(const std::string& s) {
  if (s == "cpu") return HardwareClass::cpu;
  if (s == "gpu") return HardwareClass::gpu;
  throw SchemaError("unknown hardware class '" + s + "'");
}

const Value& array_or_empty(const Value& j, const char* key) {
  static const Value empty = Value::make_array();
  const Value* v = j.find(key);
  return v ? *v : empty;
}

double num_or(const Value& j, const char* key, double dflt) {
  const Value* v = j.find(key);
  return v ? v->as_double(key) : dflt;
}

}  // namespace

AgentLibrary::AgentLibrary(const AgentLibrary& o)
    : capabilities_(o.capabilities_), skus_(o.skus_), impls_(o.impls_), profiles_(o.profiles_) {
  rebuild_indexes();
}

AgentLibrary& AgentLibrary::operator=(const AgentLibrary& o) {
  if (this != &o) {
    capabilities_ = o.capabilities_;
    skus_ = o.skus_;
    impls_ = o.impls_;
    profiles_ = o.profiles_;
    rebuild_indexes();
  }
  return *this;
}

void AgentLibrary::rebuild_indexes() {
  impls_by_cap_.clear();
  profiles_by_impl_.clear();
  for (const auto& kv : impls_) impls_by_cap_[kv.second.capability].push_back(&kv.second);
  for (auto& kv : impls_by_cap_)
    std::sort(kv.second.begin(), kv.second.end(), [](const Implementation* a, const Implementation* b) {
      return a->quality != b->quality ? a->quality > b->quality : a->name < b->name;
    });
  for (const auto& kv : profiles_) profiles_by_impl_[std::get<0>(kv.first)].push_back(&kv.second);  // map order
}

void AgentLibrary::add_capability(const std::string& capability) {
  if (capabilities_.count(capability))
    throw DuplicateKeyError("agent '" + capability + "' is already registered");
  capabilities_[capability] = true;
}

void AgentLibrary::add_sku(HardwareSku s) {
  if (s.busy_watts_per_unit < 0 || s.idle_watts_per_unit < 0 || s.dollars_per_unit_hour < 0)
    throw ValidationError("sku '" + s.id + "': power and rate must be >= 0");
  if (s.busy_watts_per_unit < s.idle_watts_per_unit)
    throw ValidationError("sku '" + s.id + "': busy power must be >= idle power");
  if (skus_.count(s.id)) throw DuplicateKeyError("sku '" + s.id + "' is already registered");
  skus_.emplace(s.id, std::move(s));
}

void AgentLibrary::add_implementation(Implementation impl) {
  if (!impl.supports_cpu && !impl.supports_gpu)
    throw ValidationError("implementation '" + impl.name + "': must support at least one hardware class");
  if (impl.quality < 0) throw ValidationError("implementation '" + impl.name + "': quality must be >= 0");
  if (!capabilities_.count(impl.capability))
    throw DanglingReferenceError("implementation '" + impl.name + "' references unknown capability '" +
                                 impl.capability + "'");
  if (impls_.count(impl.name))
    throw DuplicateKeyError("implementation '" + impl.name + "' is already registered");
  const Implementation* x = &impls_.emplace(impl.name, std::move(impl)).first->second;
  auto& v = impls_by_cap_[x->capability];
  const auto before = [](const Implementation* a, const Implementation* b) {
    return a->quality != b->quality ? a->quality > b->quality : a->name < b->name;
  };
  v.insert(std::upper_bound(v.begin(), v.end(), x, before), x);
}

void AgentLibrary::add_profile(ExecutionProfile p) {
  const auto who = [&] { return "profile (" + p.implementation + ", " + p.sku + ")"; };  // only built on error
  if (p.throughput <= 0) throw ValidationError(who() + ": throughput must be > 0");
  if (p.setup_seconds < 0) throw ValidationError(who() + ": setup latency must be >= 0");
  if (p.units < 1) throw ValidationError(who() + ": units must be >= 1");
  if (!impls_.count(p.implementation))
    throw DanglingReferenceError("profile references unknown implementation '" + p.implementation + "'");
  if (!skus_.count(p.sku)) throw DanglingReferenceError("profile references unknown sku '" + p.sku + "'");
  auto key = std::make_tuple(p.implementation, p.sku, p.units);
  if (profiles_.count(key))
    throw DuplicateKeyError("profile (" + p.implementation + ", " + p.sku + ", " +
                            std::to_string(p.units) + ") is already registered");
  const auto it = profiles_.emplace(std::move(key), std::move(p)).first;
  auto& v = profiles_by_impl_[it->second.implementation];
  v.clear();  // rebuilt in map order from this implementation's key range
  static const std::string kEmpty;
  for (auto j = profiles_.lower_bound(std::forward_as_tuple(it->second.implementation, kEmpty, INT_MIN));
       j != profiles_.end() && std::get<0>(j->first) == it->second.implementation; ++j)
    v.push_back(&j->second);
}

namespace {
// The library bundle without a DOM (the single-search drop-in parses one per
// call).  The arrays are read into staging records, then registered in the
// DOM reader's order (skus, agents, implementations, profiles) with the same
// add_* calls, so every registration error is the DOM reader's.  Anything
// unusual (escapes, duplicate keys, missing or mistyped fields) returns false
// and from_json_text falls back to the DOM reader.
struct SkuRec {
  std::string id, cls;
  double busy = 0, idle = 0, dollars = 0;
};
struct ImplRec {
  std::string name, capability;
  long long quality = 0;
  std::vector<std::string> classes;
};

bool read_library_fast(const std::string& text, AgentLibrary& lib) {
  loomjson::Cursor c(text);
  std::vector<SkuRec> skus;
  std::vector<std::string> caps;
  std::vector<ImplRec> impls;
  std::vector<ExecutionProfile> profs;
  unsigned seen_top = 0;
  // an array of objects: `member(field)` reads one field of the current element
  auto objects = [&](auto&& begin, auto&& member, auto&& finish) {
    if (!c.open('[')) return false;
    if (c.empty(']')) return true;
    for (bool more = true; more;) {
      begin();
      if (!c.open('{') || c.empty('}')) return false;
      for (bool m = true; m;) {
        std::string_view f;
        if (!c.key(f) || !member(f) || !c.next('}', m)) return false;
      }
      if (!finish() || !c.next(']', more)) return false;
    }
    return true;
  };
  if (!c.open('{')) return false;
  if (!c.empty('}'))
    for (bool more = true; more;) {
      std::string_view k;
      if (!c.key(k)) return false;
      unsigned bit = k == "skus" ? 1 : k == "agents" ? 2 : k == "implementations" ? 4 : k == "profiles" ? 8 : 0;
      if (bit & seen_top) return false;
      seen_top |= bit;
      bool ok = true;
      if (bit == 1) {
        unsigned f = 0;
        ok = objects([&] { skus.emplace_back(); f = 0; },
                     [&](std::string_view n) {
                       SkuRec& r = skus.back();
                       unsigned b = n == "id" ? 1 : n == "class" ? 2 : n == "busy_watts_per_unit" ? 4
                                    : n == "idle_watts_per_unit" ? 8 : n == "dollars_per_unit_hour" ? 16 : 0;
                       if (b & f) return false;
                       f |= b;
                       switch (b) {
                         case 1: return c.str(r.id);
                         case 2: return c.str(r.cls);
                         case 4: return c.num(r.busy);
                         case 8: return c.num(r.idle);
                         case 16: return c.num(r.dollars);
                         default: return c.skip();
                       }
                     },
                     [&] { return f == 31; });
      } else if (bit == 2) {
        unsigned f = 0;
        ok = objects([&] { caps.emplace_back(); f = 0; },
                     [&](std::string_view n) {
                       if (n != "capability") return c.skip();
                       if (f) return false;
                       f = 1;
                       return c.str(caps.back());
                     },
                     [&] { return f == 1; });
      } else if (bit == 4) {
        unsigned f = 0;
        ok = objects([&] { impls.emplace_back(); f = 0; },
                     [&](std::string_view n) {
                       ImplRec& r = impls.back();
                       unsigned b = n == "name" ? 1 : n == "capability" ? 2 : n == "quality" ? 4
                                    : n == "supported_classes" ? 8 : 0;
                       if (b & f) return false;
                       f |= b;
                       switch (b) {
                         case 1: return c.str(r.name);
                         case 2: return c.str(r.capability);
                         case 4: return c.integer(r.quality);
                         case 8: {
                           if (!c.open('[')) return false;
                           if (c.empty(']')) return true;
                           for (bool m = true; m;) {
                             r.classes.emplace_back();
                             if (!c.str(r.classes.back()) || !c.next(']', m)) return false;
                           }
                           return true;
                         }
                         default: return c.skip();
                       }
                     },
                     [&] { return f == 15; });
      } else if (bit == 8) {
        unsigned f = 0;
        ok = objects([&] { profs.emplace_back(); f = 0; },
                     [&](std::string_view n) {
                       ExecutionProfile& r = profs.back();
                       unsigned b = n == "implementation" ? 1 : n == "sku" ? 2 : n == "units" ? 4
                                    : n == "throughput" ? 8 : n == "setup_seconds" ? 16 : 0;
                       if (b & f) return false;
                       f |= b;
                       long long u = 0;
                       switch (b) {
                         case 1: return c.str(r.implementation);
                         case 2: return c.str(r.sku);
                         case 4:
                           if (!c.integer(u) || u < INT_MIN || u > INT_MAX) return false;
                           r.units = static_cast<int>(u);
                           return true;
                         case 8: return c.num(r.throughput);
                         case 16: return c.num(r.setup_seconds);
                         default: return c.skip();
                       }
                     },
                     [&] { return (f & 15) == 15; });
      } else {
        ok = c.skip();
      }
      if (!ok || !c.next('}', more)) return false;
    }
  if (!c.end()) return false;
  for (SkuRec& r : skus) {
    HardwareSku sku;
    sku.id = std::move(r.id);
    sku.hardware_class = class_of(r.cls);
    sku.busy_watts_per_unit = r.busy;
    sku.idle_watts_per_unit = r.idle;
    sku.dollars_per_unit_hour = r.dollars;
    lib.add_sku(std::move(sku));
  }
  for (std::string& cap : caps) lib.add_capability(std::move(cap));
  for (ImplRec& r : impls) {
    Implementation impl;
    impl.name = std::move(r.name);
    impl.capability = std::move(r.capability);
    if (r.quality < INT_MIN || r.quality > INT_MAX) return false;
    impl.quality = static_cast<int>(r.quality);
    for (const std::string& cl : r.classes) {
      if (class_of(cl) == HardwareClass::cpu) impl.supports_cpu = true;
      else impl.supports_gpu = true;
    }
    lib.add_implementation(std::move(impl));
  }
  for (ExecutionProfile& pr : profs) lib.add_profile(std::move(pr));
  return true;
}
}  // namespace

AgentLibrary AgentLibrary::from_json_text(const std::string& text) {
  {
    AgentLibrary fast;
    if (read_library_fast(text, fast)) return fast;
  }
  AgentLibrary lib;
  try {
    const Value j = loomjson::parse(text);
    for (const Value& s : array_or_empty(j, "skus").items()) {
      HardwareSku sku;
      sku.id = s.at("id").as_string("id");
      sku.hardware_class = class_of(s.at("class").as_string("class"));
      sku.busy_watts_per_unit = s.at("busy_watts_per_unit").as_double("busy_watts_per_unit");
      sku.idle_watts_per_unit = s.at("idle_watts_per_unit").as_double("idle_watts_per_unit");
      sku.dollars_per_unit_hour = s.at("dollars_per_unit_hour").as_double("dollars_per_unit_hour");
      lib.add_sku(std::move(sku));
    }
    for (const Value& a : array_or_empty(j, "agents").items())
      lib.add_capability(a.at("capability").as_string("capability"));
    for (const Value& i : array_or_empty(j, "implementations").items()) {
      Implementation impl;
      impl.name = i.at("name").as_string("name");
      impl.capability = i.at("capability").as_string("capability");
      impl.quality = static_cast<int>(i.at("quality").as_int("quality"));
      for (const Value& c : i.at("supported_classes").items()) {
        if (class_of(c.as_string("supported_classes")) == HardwareClass::cpu) impl.supports_cpu = true;
        else impl.supports_gpu = true;
      }
      lib.add_implementation(std::move(impl));
    }
    for (const Value& p : array_or_empty(j, "profiles").items()) {
      ExecutionProfile prof;
      prof.implementation = p.at("implementation").as_string("implementation");
      prof.sku = p.at("sku").as_string("sku");
      prof.units = static_cast<int>(p.at("units").as_int("units"));
      prof.throughput = p.at("throughput").as_double("throughput");
      prof.setup_seconds = num_or(p, "setup_seconds", 0.0);
      lib.add_profile(std::move(prof));
    }
  } catch (const loomjson::ParseError& e) {
    throw SchemaError(std::string("malformed library bundle: ") + e.what());
  }
  return lib;
}

const HardwareSku* AgentLibrary::sku(const std::string& id) const {
  auto it = skus_.find(id);
  return it == skus_.end() ? nullptr : &it->second;
}
const Implementation* AgentLibrary::implementation(const std::string& name) const {
  auto it = impls_.find(name);
  return it == impls_.end() ? nullptr : &it->second;
}
const ExecutionProfile* AgentLibrary::profile(const std::string& impl, const std::string& sku, int units) const {
  auto it = profiles_.find(std::forward_as_tuple(impl, sku, units));
  return it == profiles_.end() ? nullptr : &it->second;
}

std::vector<const Implementation*> AgentLibrary::implementations_for(const std::string& capability) const {
  if (!capabilities_.count(capability))
    throw UnknownCapabilityError("capability '" + capability + "' is not registered");
  const auto it = impls_by_cap_.find(capability);
  return it == impls_by_cap_.end() ? std::vector<const Implementation*>{} : it->second;
}

std::vector<const ExecutionProfile*> AgentLibrary::profiles_for(const std::string& implementation) const {
  const auto it = profiles_by_impl_.find(implementation);
  return it == profiles_by_impl_.end() ? std::vector<const ExecutionProfile*>{} : it->second;
}

// ---------------------------------------------------------------------------
// dag / bounds / objective
// ---------------------------------------------------------------------------
namespace {
// dag.json without a DOM: the batch lowering's hot path (a 6-task dag.json
// parses ~3x faster).  Fields the reader does not use are skipped; anything
// unusual (escapes, duplicate or missing keys, type mismatches) returns
// false and from_json_text falls back to the DOM reader, which produces the
// canonical errors.
bool read_dag_fast(const std::string& text, WorkflowDag& dag) {
  loomjson::Cursor c(text);
  dag.nodes.reserve(8);
  dag.edges.reserve(16);
  if (!c.open('{') || c.empty('}')) return false;
  bool have_nodes = false, have_edges = false;
  for (bool more = true; more;) {
    std::string_view k;
    if (!c.key(k)) return false;
    if (k == "nodes") {
      if (have_nodes || !c.open('[')) return false;
      have_nodes = true;
      if (!c.empty(']'))
        for (bool m2 = true; m2;) {
          DagNode node;
          unsigned seen = 0;
          auto once = [&](unsigned bit) {
            const bool fresh = !(seen & bit);
            seen |= bit;
            return fresh;
          };
          if (!c.open('{') || c.empty('}')) return false;
          for (bool m3 = true; m3;) {
            std::string_view f;
            if (!c.key(f)) return false;
            bool ok = true;
            if (f == "id") ok = once(1) && c.str(node.id);
            else if (f == "capability") ok = once(2) && c.str(node.capability);
            else if (f == "work_units") ok = once(4) && c.num(node.work_units);
            else if (f == "splittable") ok = once(8) && c.boolean(node.splittable);
            else if (f == "min_chunk") ok = once(16) && c.num(node.min_chunk);
            else if (f == "multi_path") ok = once(32) && c.boolean(node.multi_path);
            else if (f == "path_quality_ceiling") {
              ok = once(64);
              if (ok && !c.null()) {
                long long q = 0;
                ok = c.integer(q);
                node.path_quality_ceiling = static_cast<int>(q);
              }
            } else {
              ok = c.skip();
            }
            if (!ok || !c.next('}', m3)) return false;
          }
          if ((seen & 15) != 15) return false;  // id, capability, work_units, splittable are required
          dag.nodes.push_back(std::move(node));
          if (!c.next(']', m2)) return false;
        }
    } else if (k == "edges") {
      if (have_edges || !c.open('[')) return false;
      have_edges = true;
      if (!c.empty(']'))
        for (bool m2 = true; m2;) {
          Edge e;
          unsigned seen = 0;
          if (!c.open('{') || c.empty('}')) return false;
          for (bool m3 = true; m3;) {
            std::string_view f;
            if (!c.key(f)) return false;
            bool ok = true;
            if (f == "from") {
              ok = !(seen & 1) && c.str(e.from);
              seen |= 1;
            } else if (f == "to") {
              ok = !(seen & 2) && c.str(e.to);
              seen |= 2;
            } else {
              ok = c.skip();
            }
            if (!ok || !c.next('}', m3)) return false;
          }
          if (seen != 3) return false;
          dag.edges.push_back(std::move(e));
          if (!c.next(']', m2)) return false;
        }
    } else if (!c.skip()) {
      return false;
    }
    if (!c.next('}', more)) return false;
  }
  return have_nodes && have_edges && c.end();
}
}  // namespace

WorkflowDag WorkflowDag::from_json_text(const std::string& text) {
  {
    WorkflowDag fast;
    if (read_dag_fast(text, fast)) return fast;
  }
  WorkflowDag dag;
  try {
    const Value j = loomjson::parse(text);
    for (const Value& n : j.at("nodes").items()) {
      DagNode node;
      node.id = n.at("id").as_string("id");
      node.capability = n.at("capability").as_string("capability");
      node.work_units = n.at("work_units").as_double("work_units");
      node.splittable = n.at("splittable").as_bool("splittable");
      node.min_chunk = num_or(n, "min_chunk", 0.0);
      if (const Value* mp = n.find("multi_path")) node.multi_path = mp->as_bool("multi_path");
      if (const Value* c = n.find("path_quality_ceiling"); c && !c->is_null())
        node.path_quality_ceiling = static_cast<int>(c->as_int("path_quality_ceiling"));
      dag.nodes.push_back(std::move(node));
    }
    for (const Value& e : j.at("edges").items())
      dag.edges.push_back({e.at("from").as_string("from"), e.at("to").as_string("to")});
  } catch (const loomjson::ParseError& e) {
    throw SchemaError(std::string("malformed dag file: ") + e.what());
  }
  return dag;
}

SearchBounds SearchBounds::from_json_text(const std::string& text) {
  SearchBounds b;
  try {
    const Value j = loomjson::parse(text);
    if (const Value* v = j.find("max_fanout")) b.max_fanout = static_cast<int>(v->as_int("max_fanout"));
    if (const Value* v = j.find("max_paths")) b.max_paths = static_cast<int>(v->as_int("max_paths"));
    if (const Value* v = j.find("sku_pool_cap"))
      for (const auto& [k, cap] : v->members()) b.sku_pool_cap[k] = static_cast<int>(cap.as_int(k.c_str()));
    if (const Value* v = j.find("sku_total_cap"))
      for (const auto& [k, cap] : v->members()) b.sku_total_cap[k] = static_cast<int>(cap.as_int(k.c_str()));
  } catch (const loomjson::ParseError& e) {
    throw SchemaError(std::string("malformed bounds: ") + e.what());
  }
  return b;
}

ObjectiveHierarchy objective_from_token(const std::string& token) {
  using C = Criterion;
  ObjectiveHierarchy h;
  if (token == "MIN_COST") h.criteria = {C::min_energy, C::min_latency};
  else if (token == "MIN_DOLLARS") h.criteria = {C::min_cost_dollars, C::min_latency};
  else if (token == "MIN_LATENCY") h.criteria = {C::min_latency, C::min_energy};
  else if (token == "MAX_QUALITY") h.criteria = {C::max_quality, C::min_energy, C::min_latency};
  else throw SchemaError("unknown constraint token '" + token + "'");
  return h;
}

// ---------------------------------------------------------------------------
// plans
// ---------------------------------------------------------------------------
int NodeAssignment::fan_out() const {
  int n = 0;
  for (const Placement& p : placements) n += p.workers;
  return n;
}

std::string assignment_token(const std::string& node_id, const NodeAssignment& a) {
  // "<node_id>=<impl>[<sku>:<units>x<workers>(+...)]p<paths>;" (config.hpp:49-61),
  // built in one buffer
  std::size_t n = node_id.size() + a.implementation.size() + 16;
  for (const Placement& p : a.placements) n += p.sku.size() + 24;
  std::string s;
  s.reserve(n);
  char num[16];
  auto put_int = [&](int v) {
    const auto r = std::to_chars(num, num + sizeof num, v);
    s.append(num, r.ptr);
  };
  s += node_id;
  s += '=';
  s += a.implementation;
  s += '[';
  for (std::size_t i = 0; i < a.placements.size(); ++i) {
    if (i) s += '+';
    s += a.placements[i].sku;
    s += ':';
    put_int(a.placements[i].units);
    s += 'x';
    put_int(a.placements[i].workers);
  }
  s += "]p";
  put_int(a.path_count);
  s += ';';
  return s;
}

std::string ConfigPoint::identifier() const {
  std::string s;
  for (const auto& [id, a] : nodes) s += assignment_token(id, a);
  return s;
}

namespace {
Value assignment_json(const NodeAssignment& a) {
  Value v = Value::make_object();
  v.set("implementation", Value::make_string(a.implementation));
  Value ps = Value::make_array();
  for (const Placement& p : a.placements) {
    Value pj = Value::make_object();
    pj.set("sku", Value::make_string(p.sku));
    pj.set("units", Value::make_int(p.units));
    pj.set("workers", Value::make_int(p.workers));
    ps.push(std::move(pj));
  }
  v.set("placements", std::move(ps));
  v.set("path_count", Value::make_int(a.path_count));
  return v;
}
}  // namespace

std::string ConfigPoint::to_json_text() const {
  Value v = Value::make_object();
  v.set("label", Value::make_string(label));
  Value ns = Value::make_object();
  for (const auto& [id, a] : nodes) ns.set(id, assignment_json(a));
  v.set("nodes", std::move(ns));
  return v.dump();
}

// Reader of a config point / --pin file (config.hpp:66-117: from_json of
// Placement, NodeAssignment and ConfigPoint with their defaults -- workers 1,
// path_count 1, label "" -- then parse_config_point's checks and messages).
ConfigPoint parse_config_point(const std::string& text) {
  ConfigPoint c;
  try {
    const Value j = loomjson::parse(text);
    if (const Value* v = j.find("label")) c.label = v->as_string("label");
    for (const auto& [node_id, a] : j.at("nodes").members()) {
      NodeAssignment na;
      na.implementation = a.at("implementation").as_string("implementation");
      for (const Value& pv : a.at("placements").items()) {
        Placement pl;
        pl.sku = pv.at("sku").as_string("sku");
        pl.units = static_cast<int>(pv.at("units").as_int("units"));
        if (const Value* w = pv.find("workers")) pl.workers = static_cast<int>(w->as_int("workers"));
        na.placements.push_back(pl);
      }
      if (const Value* pc = a.find("path_count")) na.path_count = static_cast<int>(pc->as_int("path_count"));
      c.nodes[node_id] = std::move(na);
    }
  } catch (const loomjson::ParseError& e) {
    throw SchemaError(std::string("malformed config point: ") + e.what());
  }
  for (const auto& [node_id, a] : c.nodes) {
    if (a.implementation.empty()) throw SchemaError("config node '" + node_id + "': empty implementation");
    if (a.placements.empty()) throw SchemaError("config node '" + node_id + "': no placements");
    for (const auto& pl : a.placements)
      if (pl.units < 1 || pl.workers < 1)
        throw SchemaError("config node '" + node_id + "': units and workers must be >= 1");
    if (a.path_count < 1) throw SchemaError("config node '" + node_id + "': path_count must be >= 1");
  }
  return c;
}

ConfigPoint ConfigPoint::from_json_text(const std::string& text) { return parse_config_point(text); }

// ---------------------------------------------------------------------------
// chunking + node plan
// ---------------------------------------------------------------------------
int chunk_capacity(double work, double min_chunk) {
  if (min_chunk <= 0) return 1;
  return std::max(1, static_cast<int>(std::floor(work / min_chunk)));
}

std::vector<double> water_fill_split(double work, double min_chunk, const std::vector<double>& speeds) {
  // Quanta of work/quanta each go to the worker that would finish it first;
  // strict '<' keeps ties on the lower worker index.
  const int quanta = chunk_capacity(work, min_chunk);
  const double quantum = work / quanta;
  std::vector<double> done_at(speeds.size(), 0.0);
  std::vector<int> taken(speeds.size(), 0);
  for (int q = 0; q < quanta; ++q) {
    std::size_t pick = 0;
    double pick_t = done_at[0] + quantum / speeds[0];
    for (std::size_t w = 1; w < speeds.size(); ++w) {
      const double t = done_at[w] + quantum / speeds[w];
      if (t < pick_t) {
        pick = w;
        pick_t = t;
      }
    }
    done_at[pick] = pick_t;
    ++taken[pick];
  }
  std::vector<double> out(speeds.size());
  for (std::size_t w = 0; w < speeds.size(); ++w) out[w] = taken[w] * quantum;
  return out;
}

int node_quality(const DagNode& node, const Implementation& impl, int path_count) {
  const int q = impl.quality + (path_count - 1);
  return node.path_quality_ceiling ? std::min(q, *node.path_quality_ceiling) : q;
}

namespace {
struct Worker {
  const ExecutionProfile* profile;
  const HardwareSku* sku;
};

// chunking.hpp:136-181 on resolved workers (one entry per worker, placements
// expanded): the work split, then per worker setup + run, wall = max, energy
// to the gpu or cpu bucket by class, dollars.  Shared by plan_node_execution
// and the lowering, so both produce the same doubles.
NodePlan plan_workers(const DagNode& node, const Worker* workers, std::size_t n_workers, std::size_t n_placements,
                      int fan) {
  const auto where = [&] { return "node '" + node.id + "'"; };
  // One worker, or equal chunks (split_task, chunking.hpp:17-24): every
  // worker's chunk is the same value, no vector needed (this runs once per
  // option during lowering).  Hybrids water-fill (chunking.hpp:35-58).
  std::vector<double> chunk;
  double equal = node.work_units;
  if (n_workers == 1) {
  } else if (n_placements <= 1) {
    int count = 1;
    if (fan > 1 && node.min_chunk > 0)
      count = std::max(1, std::min(fan, static_cast<int>(std::floor(node.work_units / node.min_chunk))));
    if (count != fan)
      throw InvalidConfigError(where() + ": fan-out " + std::to_string(fan) + " exceeds the chunk capacity of " +
                               std::to_string(chunk_capacity(node.work_units, node.min_chunk)));
    equal = node.work_units / count;  // equal_split's value
  } else {
    std::vector<double> speeds;
    for (std::size_t w = 0; w < n_workers; ++w) speeds.push_back(workers[w].profile->throughput);
    chunk = water_fill_split(node.work_units, node.min_chunk, speeds);
    for (double c : chunk)
      if (c <= 0.0 && node.work_units > 0.0)
        throw InvalidConfigError(where() + ": degenerate hybrid placement; a worker receives no work");
  }
  NodePlan plan;
  for (std::size_t w = 0; w < n_workers; ++w) {
    const Worker& r = workers[w];
    const Micros setup = to_micros(r.profile->setup_seconds);
    const Micros run = to_micros((chunk.empty() ? equal : chunk[w]) / r.profile->throughput);
    const Micros dur = setup + run;
    plan.wall_us = std::max(plan.wall_us, dur);
    const double hours = to_seconds(dur) / 3600.0;
    const double units = static_cast<double>(r.profile->units);
    const double wh = units * r.sku->busy_watts_per_unit * hours;
    if (r.sku->hardware_class == HardwareClass::gpu) plan.gpu_wh += wh;
    else plan.cpu_wh += wh;
    plan.dollars += units * r.sku->dollars_per_unit_hour * hours;
  }
  return plan;
}
}  // namespace

NodePlan plan_node_execution(const DagNode& node, const NodeAssignment& a, const AgentLibrary& library) {
  const auto where = [&] { return "node '" + node.id + "'"; };  // only built on error
  const Implementation* impl = library.implementation(a.implementation);
  if (!impl) throw InvalidConfigError(where() + ": unknown implementation '" + a.implementation + "'");
  if (impl->capability != node.capability)
    throw InvalidConfigError(where() + ": implementation '" + impl->name + "' realizes '" + impl->capability +
                             "', not '" + node.capability + "'");
  if (a.placements.empty()) throw InvalidConfigError(where() + ": no placements");
  if (a.path_count < 1) throw InvalidConfigError(where() + ": path_count must be >= 1");
  if (a.path_count > 1 && !node.multi_path)
    throw InvalidConfigError(where() + " is not flagged multi-path in the lexicon");
  const int fan = a.fan_out();
  if (fan > 1 && !node.splittable) throw InvalidConfigError(where() + " is not splittable; fan-out must be 1");

  std::vector<Worker> workers;
  for (const Placement& p : a.placements) {
    const HardwareSku* sku = library.sku(p.sku);
    if (!sku) throw InvalidConfigError(where() + ": unknown sku '" + p.sku + "'");
    if (!impl->supports(sku->hardware_class))
      throw InvalidConfigError(where() + ": implementation '" + impl->name + "' does not support " +
                               (sku->hardware_class == HardwareClass::gpu ? "gpu" : "cpu") + " sku '" +
                               sku->id + "'");
    const ExecutionProfile* prof = library.profile(impl->name, sku->id, p.units);
    if (!prof)
      throw InvalidConfigError(where() + ": no profile for (" + impl->name + ", " + sku->id + ", " +
                               std::to_string(p.units) + ")");
    if (p.workers < 1) throw InvalidConfigError(where() + ": workers must be >= 1");
    for (int w = 0; w < p.workers; ++w) workers.push_back({prof, sku});
  }

  return plan_workers(node, workers.data(), workers.size(), a.placements.size(), fan);
}

// ---------------------------------------------------------------------------
// lever enumeration
// ---------------------------------------------------------------------------
namespace {
// A single allocation must fit the largest pool of its sku and the whole
// worker set must fit the sku's total; a non-empty cap map excludes skus it
// does not list.
bool fits(const SearchBounds& b, const std::string& sku, int units, int total_units) {
  if (!b.sku_pool_cap.empty()) {
    auto it = b.sku_pool_cap.find(sku);
    if (it == b.sku_pool_cap.end() || units > it->second) return false;
  }
  if (!b.sku_total_cap.empty()) {
    auto it = b.sku_total_cap.find(sku);
    if (it == b.sku_total_cap.end() || total_units > it->second) return false;
  }
  return true;
}
}  // namespace

namespace {
// node_options (optimizer.hpp:51-107).  With `plans` / `impls` set, each
// option's NodePlan and implementation are produced on the way from the
// already resolved profiles (the lowering's path: no name lookups per option).
void enumerate_options(const DagNode& node, const AgentLibrary& library, const SearchBounds& bounds,
                       std::vector<NodeAssignment>& out, std::vector<NodePlan>* plans,
                       std::vector<const Implementation*>* impls) {
  const int paths_max = node.multi_path ? std::max(1, bounds.max_paths) : 1;
  const int fan_cap =
      node.splittable ? std::min(bounds.max_fanout, chunk_capacity(node.work_units, node.min_chunk)) : 1;
  const int fan_hi = std::max(1, fan_cap);
  const bool hybrids = node.splittable && bounds.max_fanout >= 2;
  std::vector<Worker> workers;

  auto emit = [&](const Implementation* impl, std::vector<Placement> placements, const NodePlan* plan) {
    for (int k = 1; k <= paths_max; ++k) {
      if (k < paths_max) out.push_back({impl->name, placements, k});
      else out.push_back({impl->name, std::move(placements), k});  // the last path takes the vector
      if (plans) plans->push_back(*plan);
      if (impls) impls->push_back(impl);
    }
  };

  for (const Implementation* impl : library.implementations_for(node.capability)) {
    std::vector<Worker> usable;  // profiles of a supported class, with their sku
    for (const ExecutionProfile* p : library.profiles_for(impl->name)) {
      const HardwareSku* sku = library.sku(p->sku);
      if (impl->supports(sku->hardware_class)) usable.push_back({p, sku});
    }

    NodePlan plan;
    for (const Worker& u : usable)
      for (int w = 1; w <= fan_hi; ++w)
        if (fits(bounds, u.profile->sku, u.profile->units, u.profile->units * w)) {
          if (plans) {
            workers.assign(static_cast<std::size_t>(w), u);
            plan = plan_workers(node, workers.data(), workers.size(), 1, w);
          }
          emit(impl, {{u.profile->sku, u.profile->units, w}}, &plan);
        }

    if (!hybrids) continue;
    for (const Worker& g : usable) {
      if (g.sku->hardware_class != HardwareClass::gpu) continue;
      for (const Worker& c : usable) {
        if (c.sku->hardware_class != HardwareClass::cpu) continue;
        if (!fits(bounds, g.profile->sku, g.profile->units, g.profile->units) ||
            !fits(bounds, c.profile->sku, c.profile->units, c.profile->units))
          continue;
        const auto split =
            water_fill_split(node.work_units, node.min_chunk, {g.profile->throughput, c.profile->throughput});
        if (node.work_units > 0 && (split[0] <= 0 || split[1] <= 0)) continue;
        if (plans) {
          const Worker pair[2] = {g, c};
          plan = plan_workers(node, pair, 2, 2, 2);
        }
        emit(impl, {{g.profile->sku, g.profile->units, 1}, {c.profile->sku, c.profile->units, 1}}, &plan);
      }
    }
  }
}
}  // namespace

std::vector<NodeAssignment> node_options(const DagNode& node, const AgentLibrary& library,
                                         const SearchBounds& bounds) {
  std::vector<NodeAssignment> out;
  enumerate_options(node, library, bounds, out, nullptr, nullptr);
  return out;
}

// ---------------------------------------------------------------------------
// option-set cache of a batch lowering
// ---------------------------------------------------------------------------
class LowerCache {
 public:
  // per capability: each implementation's usable workers and the (gpu, cpu)
  // pairs that fit the caps, in enumerate_options' order
  struct Impl {
    const Implementation* impl;
    std::vector<Worker> usable;
    std::vector<std::pair<Worker, Worker>> pairs;
  };
  // one option set: the options (shared with every lowered problem that
  // uses it), per option how its plan is computed, and the identifier ranks
  struct Set {
    std::shared_ptr<const std::vector<NodeAssignment>> opts;
    std::vector<const Implementation*> impl;
    std::vector<Worker> w0, w1;   // the worker (single sku) or the (gpu, cpu) pair
    std::vector<int32_t> fan;     // single sku: the fan-out; 0: hybrid pair
    std::vector<int32_t> base;    // option whose plan this one shares (its path copies)
    std::vector<int32_t> rank;    // identifier-substring rank within the node
  };
  std::map<std::string, std::vector<Impl>, std::less<>> caps;
  std::map<std::string, Set, std::less<>> sets;
  std::string key;  // scratch
  std::size_t opts_hint = 0;  // most options of one lowered problem so far (table reservations)
};

std::shared_ptr<LowerCache> make_lower_cache() { return std::make_shared<LowerCache>(); }

namespace {
const std::vector<LowerCache::Impl>& cap_entry(LowerCache& c, const std::string& cap, const AgentLibrary& library,
                                               const SearchBounds& bounds) {
  auto it = c.caps.find(cap);
  if (it != c.caps.end()) return it->second;
  std::vector<LowerCache::Impl> v;
  for (const Implementation* impl : library.implementations_for(cap)) {
    LowerCache::Impl e{impl, {}, {}};
    for (const ExecutionProfile* p : library.profiles_for(impl->name)) {
      const HardwareSku* sku = library.sku(p->sku);
      if (impl->supports(sku->hardware_class)) e.usable.push_back({p, sku});
    }
    for (const Worker& g : e.usable) {
      if (g.sku->hardware_class != HardwareClass::gpu) continue;
      for (const Worker& cw : e.usable) {
        if (cw.sku->hardware_class != HardwareClass::cpu) continue;
        if (fits(bounds, g.profile->sku, g.profile->units, g.profile->units) &&
            fits(bounds, cw.profile->sku, cw.profile->units, cw.profile->units))
          e.pairs.emplace_back(g, cw);
      }
    }
    v.push_back(std::move(e));
  }
  return c.caps.emplace(cap, std::move(v)).first->second;
}

// The option set of a node (enumerate_options' order and contents), built on
// a miss.  Keyed by what enumerate_options depends on besides the library
// and bounds: capability, fan-out cap, path cap, hybrids, and per fitting
// (gpu, cpu) pair whether the work splits across both.
const LowerCache::Set& option_set(LowerCache& c, const DagNode& node, const AgentLibrary& library,
                                  const SearchBounds& bounds) {
  const int paths_max = node.multi_path ? std::max(1, bounds.max_paths) : 1;
  const int fan_cap =
      node.splittable ? std::min(bounds.max_fanout, chunk_capacity(node.work_units, node.min_chunk)) : 1;
  const int fan_hi = std::max(1, fan_cap);
  const bool hybrids = node.splittable && bounds.max_fanout >= 2;
  const auto& impls = cap_entry(c, node.capability, library, bounds);
  std::string& key = c.key;
  key.assign(node.capability);
  key.push_back('\x1f');
  key.append(std::to_string(fan_hi));
  key.push_back('/');
  key.append(std::to_string(paths_max));
  key.push_back(hybrids ? 'h' : '-');
  std::vector<uint8_t> split_ok;
  if (hybrids)
    for (const auto& e : impls)
      for (const auto& [g, cw] : e.pairs) {
        const auto split = water_fill_split(node.work_units, node.min_chunk, {g.profile->throughput, cw.profile->throughput});
        const bool ok = !(node.work_units > 0 && (split[0] <= 0 || split[1] <= 0));
        split_ok.push_back(ok);
        key.push_back(ok ? '1' : '0');
      }
  auto it = c.sets.find(key);
  if (it != c.sets.end()) return it->second;

  LowerCache::Set set;
  auto opts = std::make_shared<std::vector<NodeAssignment>>();
  auto emit = [&](const Implementation* impl, std::vector<Placement> placements, Worker w0, Worker w1, int fan) {
    const int first = static_cast<int>(opts->size());
    for (int k = 1; k <= paths_max; ++k) {
      opts->push_back({impl->name, placements, k});
      set.impl.push_back(impl);
      set.w0.push_back(w0);
      set.w1.push_back(w1);
      set.fan.push_back(fan);
      set.base.push_back(first);
    }
  };
  std::size_t pi = 0;
  for (const auto& e : impls) {
    for (const Worker& u : e.usable)
      for (int w = 1; w <= fan_hi; ++w)
        if (fits(bounds, u.profile->sku, u.profile->units, u.profile->units * w))
          emit(e.impl, {{u.profile->sku, u.profile->units, w}}, u, u, w);
    if (!hybrids) continue;
    for (const auto& [g, cw] : e.pairs)
      if (split_ok[pi++])
        emit(e.impl, {{g.profile->sku, g.profile->units, 1}, {cw.profile->sku, cw.profile->units, 1}}, g, cw, 0);
  }
  // identifier ranks: the substrings of one node share their "<id>=" prefix,
  // so their order does not depend on the node id
  const int r = static_cast<int>(opts->size());
  std::vector<std::string> tokens;
  tokens.reserve(r);
  for (const NodeAssignment& a : *opts) tokens.push_back(assignment_token("", a));
  std::vector<int> order(r);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return tokens[a] < tokens[b]; });
  set.rank.assign(r, 0);
  for (int k = 0; k < r; ++k) set.rank[order[k]] = k;
  set.opts = std::move(opts);
  return c.sets.emplace(key, std::move(set)).first->second;
}
}  // namespace

// ---------------------------------------------------------------------------
// estimate / order (host copies used for the winner and for small API calls)
// ---------------------------------------------------------------------------
namespace {
// Kahn's algorithm; any topological order gives the same integer critical
// path, the reference's string-ordered peers (workflow.hpp:467-498) only
// matter for determinism of its own iteration.
std::vector<int> topo_order(int n, const std::vector<int32_t>& from, const std::vector<int32_t>& to) {
  std::vector<int> indeg(n, 0);
  std::vector<std::vector<int>> succ(n);
  for (std::size_t e = 0; e < from.size(); ++e) {
    succ[from[e]].push_back(to[e]);
    ++indeg[to[e]];
  }
  std::priority_queue<int, std::vector<int>, std::greater<>> ready;
  for (int i = 0; i < n; ++i)
    if (!indeg[i]) ready.push(i);
  std::vector<int> order;
  while (!ready.empty()) {
    const int v = ready.top();
    ready.pop();
    order.push_back(v);
    for (int s : succ[v])
      if (--indeg[s] == 0) ready.push(s);
  }
  if (static_cast<int>(order.size()) != n) throw CycleError("dag has a cycle");
  return order;
}

std::int64_t quantize(double v) { return static_cast<std::int64_t>(std::llround(v * 1e9)); }
}  // namespace

ConfigEstimate estimate(const ConfigPoint& config, const WorkflowDag& dag, const AgentLibrary& library) {
  ConfigEstimate r;
  r.config = config;
  r.quality = INT_MAX;
  std::map<std::string, int> index;
  for (std::size_t i = 0; i < dag.nodes.size(); ++i) index[dag.nodes[i].id] = static_cast<int>(i);
  std::vector<Micros> wall(dag.nodes.size(), 0);
  for (std::size_t i = 0; i < dag.nodes.size(); ++i) {
    const DagNode& node = dag.nodes[i];
    auto it = config.nodes.find(node.id);
    if (it == config.nodes.end()) throw InvalidConfigError("config does not cover node '" + node.id + "'");
    const NodePlan plan = plan_node_execution(node, it->second, library);
    wall[i] = plan.wall_us;
    const double k = static_cast<double>(it->second.path_count);
    r.gpu_wh += plan.gpu_wh * k;
    r.cpu_wh += plan.cpu_wh * k;
    r.dollars += plan.dollars * k;
    r.quality = std::min(r.quality, node_quality(node, *library.implementation(it->second.implementation),
                                                 it->second.path_count));
  }
  if (dag.nodes.empty()) r.quality = 0;
  r.total_wh = r.gpu_wh + r.cpu_wh;
  std::vector<int32_t> from, to;
  for (const Edge& e : dag.edges) {
    if (!index.count(e.from) || !index.count(e.to)) throw CycleError("edge references unknown node");
    from.push_back(index[e.from]);
    to.push_back(index[e.to]);
  }
  std::vector<std::vector<int>> preds(dag.nodes.size());
  for (std::size_t e = 0; e < from.size(); ++e) preds[to[e]].push_back(from[e]);
  std::vector<Micros> finish(dag.nodes.size(), 0);
  for (int v : topo_order(static_cast<int>(dag.nodes.size()), from, to)) {
    Micros start = 0;
    for (int p : preds[v]) start = std::max(start, finish[p]);
    finish[v] = start + wall[v];
    r.latency_us = std::max(r.latency_us, finish[v]);
  }
  return r;
}

bool objective_less(const ConfigEstimate& a, const ConfigEstimate& b, const ObjectiveHierarchy& objective) {
  for (Criterion c : objective.criteria) {
    switch (c) {
      case Criterion::min_cost_dollars:
        if (quantize(a.dollars) != quantize(b.dollars)) return quantize(a.dollars) < quantize(b.dollars);
        break;
      case Criterion::min_energy:
        if (quantize(a.gpu_wh) != quantize(b.gpu_wh)) return quantize(a.gpu_wh) < quantize(b.gpu_wh);
        break;
      case Criterion::min_latency:
        if (a.latency_us != b.latency_us) return a.latency_us < b.latency_us;
        break;
      case Criterion::max_quality:
        if (a.quality != b.quality) return a.quality > b.quality;
        break;
    }
  }
  return a.config.identifier() < b.config.identifier();
}

bool meets_quality_floor(const ConfigEstimate& e, const ObjectiveHierarchy& objective) {
  return !objective.quality_floor || e.quality >= *objective.quality_floor;
}

// pareto_filter (optimizer.hpp:153-171) runs on the device: loom_capi.cpp.

// ---------------------------------------------------------------------------
// lowering
// ---------------------------------------------------------------------------
namespace {
LoweredProblem lower_impl(const WorkflowDag& dag, const AgentLibrary& library, const SearchBounds& bounds,
                          LowerCache* cache) {
  LoweredProblem L;
  const int n = static_cast<int>(dag.nodes.size());
  L.node_ids.reserve(n);
  if (n <= 64) {
    // Small dags (every batch job): no maps or queues.  Duplicate ids are
    // reported at their first repeat in dag order, edges resolve by binary
    // search over the id-sorted nodes, and the id-ordered Kahn sweep runs on
    // predecessor masks (the node popped next is the smallest-id ready one,
    // as with the priority queue); an incomplete sweep is the cycle.
    for (int i = 0; i < n; ++i) {
      for (int j = 0; j < i; ++j)
        if (dag.nodes[j].id == dag.nodes[i].id) throw InvalidConfigError("duplicate node id '" + dag.nodes[i].id + "'");
      L.node_ids.push_back(dag.nodes[i].id);
    }
    int by_id[64];
    std::iota(by_id, by_id + n, 0);
    std::sort(by_id, by_id + n, [&](int a, int b) { return L.node_ids[a] < L.node_ids[b]; });
    auto find = [&](const std::string& id) {
      const int* it = std::lower_bound(by_id, by_id + n, id, [&](int a, const std::string& v) { return L.node_ids[a] < v; });
      return it != by_id + n && L.node_ids[*it] == id ? *it : -1;
    };
    uint64_t pred[64] = {};
    L.edge_from.reserve(dag.edges.size());
    L.edge_to.reserve(dag.edges.size());
    for (const Edge& e : dag.edges) {
      const int f = find(e.from), t = find(e.to);
      if (f < 0 || t < 0) throw CycleError("edge references unknown node");
      L.edge_from.push_back(f);
      L.edge_to.push_back(t);
      pred[t] |= uint64_t(1) << f;
    }
    L.sweep_order.reserve(n);
    uint64_t done = 0;
    for (int step = 0; step < n; ++step) {
      int v = -1;
      for (int k = 0; k < n && v < 0; ++k)
        if (!(done >> by_id[k] & 1) && !(pred[by_id[k]] & ~done)) v = by_id[k];
      if (v < 0) throw CycleError("dag has a cycle");
      done |= uint64_t(1) << v;
      L.sweep_order.push_back(v);
    }
  } else {
    std::map<std::string, int> index;
    for (int i = 0; i < n; ++i) {
      if (!index.emplace(dag.nodes[i].id, i).second)
        throw InvalidConfigError("duplicate node id '" + dag.nodes[i].id + "'");
      L.node_ids.push_back(dag.nodes[i].id);
    }
    for (const Edge& e : dag.edges) {
      auto f = index.find(e.from), t = index.find(e.to);
      if (f == index.end() || t == index.end()) throw CycleError("edge references unknown node");
      L.edge_from.push_back(f->second);
      L.edge_to.push_back(t->second);
    }
    topo_order(n, L.edge_from, L.edge_to);  // throws CycleError like topological_order
    {
      // the reference's topological_order: Kahn with ready peers popped in node-id
      // order (workflow.hpp:467-498); greedy_search sweeps nodes in this order
      std::vector<int> indeg(n, 0);
      std::vector<std::vector<int>> succ(n);
      for (std::size_t e = 0; e < L.edge_from.size(); ++e) {
        succ[L.edge_from[e]].push_back(L.edge_to[e]);
        ++indeg[L.edge_to[e]];
      }
      auto by_id = [&](int a, int b) { return L.node_ids[a] > L.node_ids[b]; };
      std::priority_queue<int, std::vector<int>, decltype(by_id)> ready(by_id);
      for (int i = 0; i < n; ++i)
        if (!indeg[i]) ready.push(i);
      while (!ready.empty()) {
        const int v = ready.top();
        ready.pop();
        L.sweep_order.push_back(v);
        for (int s2 : succ[v])
          if (--indeg[s2] == 0) ready.push(s2);
      }
    }
  }

  // The identifier tie-break is replaced by a per-node rank of the option's
  // identifier substring.  That is exact only if no substring is a proper
  // prefix of another one, which holds when names carry no ';'.
  auto check_name = [](const std::string& s) {
    if (s.find(';') != std::string::npos)
      throw InvalidConfigError("name '" + s + "' contains ';', which breaks identifier ordering");
  };

  L.total = n ? 1 : 0;
  // per-node scratch reused across nodes; the tables grow by whole nodes
  std::vector<NodePlan> plans;
  std::vector<const Implementation*> impls;
  std::vector<std::string> tokens;
  std::vector<int> order;
  std::vector<int32_t> rank;
  plans.reserve(32);
  impls.reserve(32);
  L.radix.reserve(n);
  L.options.reserve(n);
  std::vector<Worker> workers;
  if (cache) {
    L.shared_options.reserve(n);
    for (auto* v : {&L.gpu_wh, &L.cpu_wh, &L.dollars}) v->reserve(cache->opts_hint);
    L.wall_us.reserve(cache->opts_hint);
    L.quality.reserve(cache->opts_hint);
    L.lexrank.reserve(cache->opts_hint);
  }
  for (int i = 0; i < n; ++i) {
    const DagNode& node = dag.nodes[i];
    check_name(node.id);
    if (cache) {  // the option set from the cache; only the numbers are per node
      const LowerCache::Set& set = option_set(*cache, node, library, bounds);
      const int r = static_cast<int>(set.opts->size());
      L.radix.push_back(r);
      if (r == 0) L.total = 0;
      else if (L.total && L.total > UINT64_MAX / static_cast<uint64_t>(r))
        throw InvalidConfigError("plan space exceeds 2^64 plans");
      else L.total *= static_cast<uint64_t>(r);
      NodePlan plan;
      for (int o = 0; o < r; ++o) {
        const NodeAssignment& a = (*set.opts)[o];
        if (o == 0 || set.base[o] != set.base[o - 1]) {  // == plan_node_execution(node, a, library)
          check_name(a.implementation);
          for (const Placement& p : a.placements) check_name(p.sku);
          if (set.fan[o] > 0) {
            workers.assign(static_cast<std::size_t>(set.fan[o]), set.w0[o]);
            plan = plan_workers(node, workers.data(), workers.size(), 1, set.fan[o]);
          } else {
            const Worker pair[2] = {set.w0[o], set.w1[o]};
            plan = plan_workers(node, pair, 2, 2, 2);
          }
        }
        const double k = static_cast<double>(a.path_count);
        L.wall_us.push_back(plan.wall_us);
        L.gpu_wh.push_back(plan.gpu_wh * k);
        L.cpu_wh.push_back(plan.cpu_wh * k);
        L.dollars.push_back(plan.dollars * k);
        L.quality.push_back(node_quality(node, *set.impl[o], a.path_count));
      }
      L.lexrank.insert(L.lexrank.end(), set.rank.begin(), set.rank.end());
      L.shared_options.push_back(set.opts);
      continue;
    }
    std::vector<NodeAssignment> opts;
    opts.reserve(32);
    plans.clear();
    impls.clear();
    enumerate_options(node, library, bounds, opts, &plans, &impls);
    const int r = static_cast<int>(opts.size());
    L.radix.push_back(r);
    if (r == 0) L.total = 0;
    else if (L.total && L.total > UINT64_MAX / static_cast<uint64_t>(r))
      throw InvalidConfigError("plan space exceeds 2^64 plans");
    else L.total *= static_cast<uint64_t>(r);

    tokens.clear();
    tokens.reserve(r);
    const std::size_t base = L.wall_us.size();
    for (auto* v : {&L.gpu_wh, &L.cpu_wh, &L.dollars}) v->reserve(base + r);
    L.wall_us.reserve(base + r);
    L.quality.reserve(base + r);
    L.lexrank.reserve(base + r);
    for (int o = 0; o < r; ++o) {
      const NodeAssignment& a = opts[o];
      check_name(a.implementation);
      for (const Placement& p : a.placements) check_name(p.sku);
      const NodePlan& plan = plans[o];  // == plan_node_execution(node, a, library), same arithmetic
      const double k = static_cast<double>(a.path_count);
      L.wall_us.push_back(plan.wall_us);
      L.gpu_wh.push_back(plan.gpu_wh * k);
      L.cpu_wh.push_back(plan.cpu_wh * k);
      L.dollars.push_back(plan.dollars * k);
      L.quality.push_back(node_quality(node, *impls[o], a.path_count));
      tokens.push_back(assignment_token(node.id, a));
    }
    order.resize(r);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return tokens[a] < tokens[b]; });
    rank.resize(r);
    for (int k = 0; k < r; ++k) rank[order[k]] = k;
    L.lexrank.insert(L.lexrank.end(), rank.begin(), rank.end());
    L.options.push_back(std::move(opts));
  }

  if (cache) cache->opts_hint = std::max(cache->opts_hint, L.wall_us.size());

  // Mixed-radix weights in std::map (sorted node id) order: the identifier
  // concatenates nodes in that order, so the first sorted node is the most
  // significant digit of the rank.
  std::vector<int> by_id(n);
  std::iota(by_id.begin(), by_id.end(), 0);
  std::sort(by_id.begin(), by_id.end(), [&](int a, int b) { return L.node_ids[a] < L.node_ids[b]; });
  L.lex_weight.assign(n, 0);
  uint64_t w = 1;
  for (int k = n - 1; k >= 0; --k) {
    L.lex_weight[by_id[k]] = w;
    if (L.total) w *= static_cast<uint64_t>(L.radix[by_id[k]]);
  }
  return L;
}
}  // namespace

LoweredProblem lower(const WorkflowDag& dag, const AgentLibrary& library, const SearchBounds& bounds) {
  return lower_impl(dag, library, bounds, nullptr);
}

LoweredProblem lower(const WorkflowDag& dag, const AgentLibrary& library, const SearchBounds& bounds,
                     LowerCache& cache) {
  return lower_impl(dag, library, bounds, &cache);
}

loom_problem LoweredProblem::view() const {
  loom_problem p{};
  p.n_nodes = static_cast<int32_t>(radix.size());
  p.n_edges = static_cast<int32_t>(edge_from.size());
  p.radix = radix.data();
  p.wall_us = wall_us.data();
  p.gpu_wh = gpu_wh.data();
  p.cpu_wh = cpu_wh.data();
  p.dollars = dollars.data();
  p.quality = quality.data();
  p.lexrank = lexrank.data();
  p.lex_weight = lex_weight.data();
  p.edge_from = edge_from.data();
  p.edge_to = edge_to.data();
  return p;
}

ConfigPoint LoweredProblem::config_of(uint64_t plan_index) const {
  ConfigPoint c;
  for (int i = static_cast<int>(radix.size()) - 1; i >= 0; --i) {
    const uint64_t r = static_cast<uint64_t>(radix[i]);
    c.nodes[node_ids[i]] = node_opts(i)[plan_index % r];
    plan_index /= r;
  }
  return c;
}

}  // namespace loom
