// CommLedger of the reference protocol: the bytes a SPES run's frames
// carry under the reference's parameter-server protocol, per (node, round), with the same
// accounting (protocol.hpp:29-52; Server::on_bytes / broadcast_global / handle,
// protocol.cpp:56-175; in-process driver run_inproc :368-405). Every frame is an 18-byte
// header plus its payload (wire.cpp:58-94); payload sizes follow the codec of wire.cpp
// (HELLO 12 B, ASSIGN 8 + 4|experts| B, blocks as encode_blocks). The B200 path moves
// these parameters over NCCL instead; the ledger keeps the reference's byte accounting.
#include <cstdint>
#include <map>
#include <stdexcept>
#include <utility>
#include <vector>

#include "wire.hpp"

namespace spes_ledger {

struct Entry {
    int32_t node, round;
    uint64_t up, down;
};

constexpr uint64_t kHeader = 18;

std::vector<Entry> expected(int64_t V, int64_t d, int64_t f, int L, int M, int nodes,
                            const std::vector<std::vector<int>>& owned, int rounds, bool diloco,
                            uint64_t totals[4]) {
    if (nodes < 1) throw std::invalid_argument("server: need at least one node");
    if (rounds < 1) throw std::invalid_argument("server: need at least one round");
    if (static_cast<int>(owned.size()) != nodes)
        throw std::invalid_argument("ledger: ownership map needs one entry per node");
    const std::vector<spes_wire::Block> all = spes_wire::model_blocks(V, d, f, L, M);
    const size_t npsi = 2 + 2 * static_cast<size_t>(L);
    const uint64_t global = kHeader + static_cast<uint64_t>(spes_wire::payload_bytes(all));
    std::map<std::pair<int, int>, std::pair<uint64_t, uint64_t>> led;
    uint64_t up = 0, down = 0, pushes = 0, broadcasts = 0;
    auto add_up = [&](int n, int r, uint64_t b) { led[{n, r}].first += b, up += b; };
    auto add_down = [&](int n, int r, uint64_t b) { led[{n, r}].second += b, down += b; };
    for (int n = 0; n < nodes; ++n) {
        add_up(-1, 0, kHeader + 12);  // HELLO: the connection has no node yet
        add_down(n, 0, kHeader + 8 + 4 * owned[n].size());  // ASSIGN
    }
    std::vector<uint64_t> update(static_cast<size_t>(nodes));
    for (int n = 0; n < nodes; ++n) {
        if (diloco) {
            update[n] = global;
            continue;
        }
        std::vector<spes_wire::Block> blocks(all.begin(), all.begin() + npsi);  // shared
        std::vector<char> mine(static_cast<size_t>(M), 0);
        for (int e : owned[n]) {
            if (e < 0 || e >= M) throw std::invalid_argument("ownership: expert id out of range");
            mine[e] = 1;
        }
        for (int l = 0; l < L; ++l)  // sparse_update_blocks: enumerate order, owned only
            for (int j = 0; j < M; ++j)
                if (mine[j])
                    for (int w = 0; w < 3; ++w)
                        blocks.push_back(all[npsi + (static_cast<size_t>(l) * M + j) * 3 + w]);
        update[n] = kHeader + static_cast<uint64_t>(spes_wire::payload_bytes(blocks));
    }
    auto broadcast = [&](int r) {
        for (int n = 0; n < nodes; ++n) add_down(n, r, global), ++broadcasts;
    };
    broadcast(1);  // once every node has joined
    for (int r = 1; r <= rounds; ++r) {
        for (int n = 0; n < nodes; ++n) {
            add_up(n, r, update[n]);  // LOCAL_UPDATE
            ++pushes;
            add_down(n, r, kHeader);  // ROUND_DONE
        }
        broadcast(r + 1);  // the next round's model, or the final one
    }
    for (int n = 0; n < nodes; ++n) add_down(n, rounds + 1, kHeader);  // BYE
    for (int n = 0; n < nodes; ++n) add_up(n, rounds + 1, kHeader);    // the workers' BYE
    std::vector<Entry> out;
    for (const auto& [k, v] : led) out.push_back({k.first, k.second, v.first, v.second});
    totals[0] = up;
    totals[1] = down;
    totals[2] = pushes;
    totals[3] = broadcasts;
    return out;
}

}  // namespace spes_ledger

#include <sstream>
#include <string>

namespace spes_ledger {

struct RoundRow {
    int32_t round;
    double mean_total, mean_ce, mean_lb, mean_moe_z, mean_z, merge_displacement_sq;
    uint64_t bytes_up, bytes_down;
};

// metrics.csv of an experiment directory (experiment.cpp:376-385): the same header, column
// order and default ostream formatting of doubles
std::string metrics_csv(const RoundRow* rows, int n, int64_t tokens_per_round,
                        const double* wall_ms, int n_wall) {
    std::ostringstream csv;
    csv << "round,tokens_seen,total,ce,lb,moe_z,z,bytes_up,bytes_down,merge_displacement_sq,"
           "wall_ms\n";
    for (int i = 0; i < n; ++i) {
        const RoundRow& m = rows[i];
        csv << m.round << ',' << tokens_per_round * m.round << ',' << m.mean_total << ','
            << m.mean_ce << ',' << m.mean_lb << ',' << m.mean_moe_z << ',' << m.mean_z << ','
            << m.bytes_up << ',' << m.bytes_down << ',' << m.merge_displacement_sq << ','
            << (i < n_wall ? wall_ms[i] : 0.0) << '\n';
    }
    return csv.str();
}

}  // namespace spes_ledger
