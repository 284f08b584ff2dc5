// Wire / checkpoint format (see wire.hpp for the reference lines each function follows).
#include "wire.hpp"

#include <cstring>
#include <fstream>
#include <iterator>
#include <unordered_set>

namespace spes_wire {

const char* proto_error_name(ProtoError e) {
    static const char* names[] = {"BadMagic",        "BadVersion",      "UnknownKind",
                                  "Truncated",       "LengthMismatch",  "MalformedPayload",
                                  "ConfigMismatch",  "RoundMismatch",   "DuplicatePush",
                                  "NotOwnedBlock",   "UnexpectedMessage", "BarrierViolation",
                                  "Timeout"};
    return names[static_cast<int>(e)];
}

std::vector<Block> model_blocks(int64_t V, int64_t d, int64_t f, int L, int M) {
    std::vector<Block> out;
    int64_t off = 0;
    auto add = [&](std::string name, std::vector<int64_t> shape) {
        int64_t n = 1;
        for (int64_t s : shape) n *= s;
        out.push_back({std::move(name), std::move(shape), off, n});
        off += n;
    };
    add("psi.emb", {V, d});
    add("psi.head", {d, V});
    for (int l = 0; l < L; ++l) {
        add("psi.norm." + std::to_string(l), {d});
        add("psi.router." + std::to_string(l), {d, M});
    }
    for (int l = 0; l < L; ++l)
        for (int j = 0; j < M; ++j) {
            const std::string base = "e." + std::to_string(l) + "." + std::to_string(j) + ".";
            add(base + "wg", {d, f});
            add(base + "wu", {d, f});
            add(base + "wd", {f, d});
        }
    return out;
}

int64_t payload_bytes(const std::vector<Block>& blocks) {
    int64_t n = 4;
    for (const auto& b : blocks)
        n += 2 + static_cast<int64_t>(b.name.size()) + 1 + 1 + 4 * static_cast<int64_t>(b.shape.size()) +
             4 * b.numel;
    return n;
}

namespace {

inline void put_u16(uint8_t*& p, uint16_t v) {
    p[0] = static_cast<uint8_t>(v & 0xff);
    p[1] = static_cast<uint8_t>(v >> 8);
    p += 2;
}
inline void put_u32(uint8_t*& p, uint32_t v) {
    for (int i = 0; i < 4; ++i) p[i] = static_cast<uint8_t>((v >> (8 * i)) & 0xff);
    p += 4;
}

struct Reader {
    const uint8_t* buf;
    size_t size;
    size_t pos = 0;
    void need(size_t n, const char* what) const {
        if (pos + n > size)
            throw ProtocolError(ProtoError::Truncated,
                                std::string("truncated payload while reading ") + what);
    }
    uint8_t u8(const char* what) {
        need(1, what);
        return buf[pos++];
    }
    uint16_t u16(const char* what) {
        need(2, what);
        const uint16_t v = static_cast<uint16_t>(buf[pos] | (buf[pos + 1] << 8));
        pos += 2;
        return v;
    }
    uint32_t u32(const char* what) {
        need(4, what);
        uint32_t v = 0;
        for (int i = 0; i < 4; ++i) v |= static_cast<uint32_t>(buf[pos + i]) << (8 * i);
        pos += 4;
        return v;
    }
};

}  // namespace

void encode_model(const std::vector<Block>& blocks, const float* params, uint8_t* out) {
    uint8_t* p = out;
    put_u32(p, static_cast<uint32_t>(blocks.size()));
    for (const auto& b : blocks) {
        put_u16(p, static_cast<uint16_t>(b.name.size()));
        std::memcpy(p, b.name.data(), b.name.size());
        p += b.name.size();
        *p++ = 0;  // dtype f32
        *p++ = static_cast<uint8_t>(b.shape.size());
        for (int64_t dim : b.shape) put_u32(p, static_cast<uint32_t>(dim));
        std::memcpy(p, params + b.offset, 4 * static_cast<size_t>(b.numel));  // little-endian host
        p += 4 * b.numel;
    }
}

void decode_model(const std::vector<Block>& blocks, const uint8_t* payload, int64_t len,
                  float* params) {
    Reader r{payload, static_cast<size_t>(len)};
    const uint32_t count = r.u32("block count");
    std::unordered_set<std::string> seen;
    struct Parsed {
        std::string name;
        std::vector<int64_t> shape;
        size_t data_pos;
    };
    std::vector<Parsed> parsed;
    for (uint32_t i = 0; i < count; ++i) {  // decode_blocks (wire.cpp:117-152)
        const uint16_t nlen = r.u16("name length");
        r.need(nlen, "block name");
        std::string name(reinterpret_cast<const char*>(payload + r.pos), nlen);
        r.pos += nlen;
        if (!seen.insert(name).second)
            throw ProtocolError(ProtoError::MalformedPayload, "duplicate block name " + name);
        const uint8_t dtype = r.u8("dtype");
        if (dtype != 0)
            throw ProtocolError(ProtoError::MalformedPayload,
                                "unsupported dtype " + std::to_string(dtype));
        const uint8_t rank = r.u8("rank");
        if (rank == 0 || rank > 4)
            throw ProtocolError(ProtoError::MalformedPayload, "bad rank for block " + name);
        std::vector<int64_t> shape;
        uint64_t numel = 1;
        for (uint8_t dd = 0; dd < rank; ++dd) {
            const uint32_t dim = r.u32("dim");
            shape.push_back(static_cast<int64_t>(dim));
            numel *= dim;
            if (numel > (1ull << 33))
                throw ProtocolError(ProtoError::MalformedPayload,
                                    "implausible element count for block " + name);
        }
        r.need(numel * 4, "block values");
        parsed.push_back({std::move(name), std::move(shape), r.pos});
        r.pos += numel * 4;
    }
    if (r.pos != r.size)
        throw ProtocolError(ProtoError::MalformedPayload, "trailing bytes after blocks");
    // blocks_into_model (wire.cpp:161-176)
    if (parsed.size() != blocks.size())
        throw ProtocolError(ProtoError::MalformedPayload,
                            "model payload block count " + std::to_string(parsed.size()) +
                                " != expected " + std::to_string(blocks.size()));
    for (size_t i = 0; i < blocks.size(); ++i)
        if (parsed[i].name != blocks[i].name || parsed[i].shape != blocks[i].shape)
            throw ProtocolError(ProtoError::MalformedPayload,
                                "unexpected block " + parsed[i].name + " at position " +
                                    std::to_string(i));
    for (size_t i = 0; i < blocks.size(); ++i)
        std::memcpy(params + blocks[i].offset, payload + parsed[i].data_pos,
                    4 * static_cast<size_t>(blocks[i].numel));
}

void write_checkpoint(const std::string& path, const std::vector<Block>& blocks,
                      const float* params, uint64_t round) {
    std::vector<uint8_t> bytes(static_cast<size_t>(payload_bytes(blocks)) + 8);
    encode_model(blocks, params, bytes.data());
    for (int i = 0; i < 8; ++i)
        bytes[bytes.size() - 8 + i] = static_cast<uint8_t>((round >> (8 * i)) & 0xff);
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    if (!f) throw std::runtime_error("cannot open checkpoint for writing: " + path);
    f.write(reinterpret_cast<const char*>(bytes.data()), static_cast<std::streamsize>(bytes.size()));
    if (!f) throw std::runtime_error("checkpoint write failed: " + path);
}

uint64_t read_checkpoint(const std::string& path, const std::vector<Block>& blocks, float* params) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot open checkpoint: " + path);
    std::vector<uint8_t> bytes((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    if (bytes.size() < 8)
        throw ProtocolError(ProtoError::Truncated, "checkpoint shorter than round trailer");
    uint64_t round = 0;
    for (int i = 0; i < 8; ++i)
        round |= static_cast<uint64_t>(bytes[bytes.size() - 8 + i]) << (8 * i);
    decode_model(blocks, bytes.data(), static_cast<int64_t>(bytes.size()) - 8, params);
    return round;
}

}  // namespace spes_wire
