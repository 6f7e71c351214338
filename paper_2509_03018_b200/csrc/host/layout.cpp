// layout.cpp — DP/PP/TP group tables and the per-iteration op program that
// config-file runs analyze against. Behaviour follows the reference's
// build_layout (proj/src/topology.cpp:80-148: comm_ids assigned DP, then PP,
// then TP; rank = dp_i*pp*tp + pp_i*tp + tp_i) and default_program
// (proj/src/program.cpp:25-119: per pipeline stage Recv, TP AllGather, Send,
// DP ReduceScatter + AllGather, chained on each rank's previous op).
#include <algorithm>
#include <deque>
#include <map>

#include "host.h"

namespace csh {

Layout build_layout(int tp, int pp, int dp, int rpn, int cpp, int nics) {
  if (tp < 1 || pp < 1 || dp < 1 || rpn < 1 || cpp < 1 || nics < 1)
    throw ConfigError("layout: all dimensions must be >= 1");
  const int world = tp * pp * dp;
  if (world % rpn != 0)
    throw ConfigError("layout: world size " + std::to_string(world) +
                      " not divisible by ranks_per_node " + std::to_string(rpn));
  if (tp > rpn)
    throw ConfigError("layout: tp " + std::to_string(tp) +
                      " exceeds ranks_per_node " + std::to_string(rpn) +
                      " (TP must stay intra-node)");
  Layout l;
  l.tp = tp;
  l.pp = pp;
  l.dp = dp;
  l.ranks_per_node = rpn;
  l.channels_per_pair = cpp;
  l.nics_per_node = nics;
  auto rank_of = [&](int d, int p, int t) { return d * (pp * tp) + p * tp + t; };
  auto add = [&](uint8_t kind, std::vector<int32_t> m) {
    l.kind.push_back(kind);
    l.members.push_back(std::move(m));
  };
  for (int p = 0; p < pp; ++p)
    for (int t = 0; t < tp; ++t) {
      std::vector<int32_t> m;
      for (int d = 0; d < dp; ++d) m.push_back(rank_of(d, p, t));
      add(CSG_GROUP_DP, std::move(m));
    }
  for (int d = 0; d < dp; ++d)
    for (int t = 0; t < tp; ++t) {
      std::vector<int32_t> m;
      for (int p = 0; p < pp; ++p) m.push_back(rank_of(d, p, t));
      add(CSG_GROUP_PP, std::move(m));
    }
  for (int d = 0; d < dp; ++d)
    for (int p = 0; p < pp; ++p) {
      std::vector<int32_t> m;
      for (int t = 0; t < tp; ++t) m.push_back(rank_of(d, p, t));
      add(CSG_GROUP_TP, std::move(m));
    }
  return l;
}

namespace {

std::vector<int32_t> executing(const Op& op, const Layout& l) {
  if (op.name == CSG_OP_SEND) return {op.src};
  if (op.name == CSG_OP_RECV) return {op.dst};
  return l.members[static_cast<size_t>(op.group)];
}

}  // namespace

Program default_program(const Layout& l, uint64_t msg_bytes) {
  if (msg_bytes == 0)
    throw ConfigError("default_program: msg_bytes must be > 0");
  Program prog;
  std::map<int32_t, int64_t> last;  // rank -> most recent op this iteration
  auto deps_of = [&](const std::vector<int32_t>& ranks) {
    std::vector<int64_t> d;
    for (int32_t r : ranks) {
      auto it = last.find(r);
      if (it != last.end()) d.push_back(it->second);
    }
    std::sort(d.begin(), d.end());
    d.erase(std::unique(d.begin(), d.end()), d.end());
    return d;
  };
  auto push = [&](Op op) {
    const int64_t seq = static_cast<int64_t>(prog.ops.size());
    for (int32_t r : executing(op, l)) last[r] = seq;
    prog.ops.push_back(std::move(op));
    return seq;
  };
  std::vector<int32_t> dpg, ppg, tpg;
  for (size_t g = 0; g < l.kind.size(); ++g) {
    if (l.kind[g] == CSG_GROUP_DP) dpg.push_back(static_cast<int32_t>(g));
    if (l.kind[g] == CSG_GROUP_PP) ppg.push_back(static_cast<int32_t>(g));
    if (l.kind[g] == CSG_GROUP_TP) tpg.push_back(static_cast<int32_t>(g));
  }
  auto stage_of = [&](int32_t rank) { return (rank / l.tp) % l.pp; };
  std::map<std::pair<int32_t, int>, int64_t> send_seq;  // (pp group, stage)
  for (int stage = 0; stage < l.pp; ++stage) {
    if (stage > 0) {
      for (int32_t g : ppg) {
        const auto& m = l.members[g];
        Op op;
        op.name = CSG_OP_RECV;
        op.group = g;
        op.src = m[stage - 1];
        op.dst = m[stage];
        const int64_t snd = send_seq.at({g, stage - 1});
        op.deps = deps_of({op.dst});
        if (std::find(op.deps.begin(), op.deps.end(), snd) == op.deps.end())
          op.deps.push_back(snd);
        std::sort(op.deps.begin(), op.deps.end());
        push(std::move(op));
      }
    }
    for (int32_t g : tpg) {
      const auto& m = l.members[g];
      if (stage_of(m.front()) != stage || m.size() < 2) continue;
      Op op;
      op.name = CSG_OP_ALLGATHER;
      op.group = g;
      op.deps = deps_of(m);
      push(std::move(op));
    }
    if (stage + 1 < l.pp) {
      for (int32_t g : ppg) {
        const auto& m = l.members[g];
        Op op;
        op.name = CSG_OP_SEND;
        op.group = g;
        op.src = m[stage];
        op.dst = m[stage + 1];
        op.deps = deps_of({op.src});
        send_seq[{g, stage}] = push(std::move(op));
      }
    }
    for (int32_t g : dpg) {
      const auto& m = l.members[g];
      if (stage_of(m.front()) != stage || m.size() < 2) continue;
      Op rs;
      rs.name = CSG_OP_REDUCESCATTER;
      rs.group = g;
      rs.deps = deps_of(m);
      const int64_t rs_seq = push(std::move(rs));
      Op ag;
      ag.name = CSG_OP_ALLGATHER;
      ag.group = g;
      ag.deps = {rs_seq};
      push(std::move(ag));
    }
  }
  validate_program(prog, l);
  return prog;
}

void validate_program(const Program& p, const Layout& l) {
  // validate_program (proj/src/program.cpp:121-145) for the checks that can
  // fail on a generated program: group ids, earlier-only deps, p2p ends.
  const size_t n = p.ops.size();
  for (size_t i = 0; i < n; ++i) {
    const Op& op = p.ops[i];
    if (op.group < 0 || static_cast<size_t>(op.group) >= l.members.size())
      throw ConfigError("unknown comm_id " + std::to_string(op.group));
    for (int64_t d : op.deps)
      if (d < 0 || d >= static_cast<int64_t>(i))
        throw ConfigError("program: op " + std::to_string(i) +
                          " depends on non-earlier op " + std::to_string(d));
    if ((op.name == CSG_OP_SEND || op.name == CSG_OP_RECV) &&
        (op.src < 0 || op.dst < 0 || op.src == op.dst))
      throw ConfigError("program: p2p op " + std::to_string(i) +
                        " needs distinct src and dst");
  }
}

Tables::Tables(const Layout& l, const Program& p) {
  kind = l.kind;
  member_off.assign(1, 0);
  for (const auto& m : l.members) {
    members.insert(members.end(), m.begin(), m.end());
    member_off.push_back(static_cast<int64_t>(members.size()));
  }
  dep_off.assign(1, 0);
  for (const Op& op : p.ops) {
    op_name.push_back(op.name);
    group.push_back(op.group);
    src.push_back(op.src);
    dst.push_back(op.dst);
    deps.insert(deps.end(), op.deps.begin(), op.deps.end());
    dep_off.push_back(static_cast<int64_t>(deps.size()));
  }
  topo.world_size = l.world();
  topo.n_groups = static_cast<int32_t>(l.members.size());
  topo.group_kind = kind.data();
  topo.member_off = member_off.data();
  topo.members = members.data();
  prog.n_ops = static_cast<int32_t>(p.ops.size());
  prog.op_name = op_name.data();
  prog.group = group.data();
  prog.src = src.data();
  prog.dst = dst.data();
  prog.dep_off = dep_off.data();
  prog.deps = deps.data();
}

std::string layout_json(const Layout& l, const Program& p) {
  std::string o = "{\"world_size\":" + std::to_string(l.world()) + ",\"groups\":[";
  for (size_t g = 0; g < l.members.size(); ++g) {
    if (g) o += ",";
    o += "{\"kind\":" + std::to_string(l.kind[g]) + ",\"members\":[";
    for (size_t i = 0; i < l.members[g].size(); ++i) {
      if (i) o += ",";
      o += std::to_string(l.members[g][i]);
    }
    o += "]}";
  }
  o += "],\"ops\":[";
  for (size_t i = 0; i < p.ops.size(); ++i) {
    const Op& op = p.ops[i];
    if (i) o += ",";
    o += "{\"name\":" + std::to_string(op.name) + ",\"group\":" +
         std::to_string(op.group) + ",\"src\":" + std::to_string(op.src) +
         ",\"dst\":" + std::to_string(op.dst) + ",\"deps\":[";
    for (size_t k = 0; k < op.deps.size(); ++k) {
      if (k) o += ",";
      o += std::to_string(op.deps[k]);
    }
    o += "]}";
  }
  return o + "]}";
}

}  // namespace csh
