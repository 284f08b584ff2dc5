// Wire / checkpoint format of the reference, host side:
//   encode_blocks / decode_blocks     proj/src/wire.cpp:96-152
//   model_to_blocks / blocks_into_model  proj/src/wire.cpp:154-176
//   write_checkpoint / read_checkpoint   proj/src/wire.cpp:212-236
// Byte layout (little-endian): u32 block count; per block u16 name length + name, u8 dtype
// (0 = f32), u8 rank + u32 dims, raw f32 values. A checkpoint is that payload followed by a
// u64 round. Blocks are the model's enumerate_blocks order (model.hpp:95-111), which is
// also the flat parameter layout of the library, so every block's values are one
// contiguous run of the parameter vector.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace spes_wire {

// ProtoError of the reference (wire.hpp:23-37); carried as the message prefix
enum class ProtoError {
    BadMagic,
    BadVersion,
    UnknownKind,
    Truncated,
    LengthMismatch,
    MalformedPayload,
    ConfigMismatch,
    RoundMismatch,
    DuplicatePush,
    NotOwnedBlock,
    UnexpectedMessage,
    BarrierViolation,
    Timeout
};
const char* proto_error_name(ProtoError e);

class ProtocolError : public std::runtime_error {
public:
    ProtocolError(ProtoError c, const std::string& what)
        : std::runtime_error(std::string("[") + proto_error_name(c) + "] " + what), code(c) {}
    ProtoError code;
};

struct Block {
    std::string name;
    std::vector<int64_t> shape;
    int64_t offset;  // in floats, in the flat parameter vector
    int64_t numel;
};

// enumerate_blocks of a model (tied_head must be 0 on this path)
std::vector<Block> model_blocks(int64_t V, int64_t d, int64_t f, int L, int M);

// bytes of encode_blocks(model_to_blocks(params))
int64_t payload_bytes(const std::vector<Block>& blocks);

// encode_blocks(model_to_blocks(params)) into out (payload_bytes bytes)
void encode_model(const std::vector<Block>& blocks, const float* params, uint8_t* out);

// decode_blocks + blocks_into_model: validates the payload exactly as the reference does
// (same error classes and messages) and writes the values into params
void decode_model(const std::vector<Block>& blocks, const uint8_t* payload, int64_t len,
                  float* params);

void write_checkpoint(const std::string& path, const std::vector<Block>& blocks,
                      const float* params, uint64_t round);
// returns the round; params receives the model
uint64_t read_checkpoint(const std::string& path, const std::vector<Block>& blocks, float* params);

}  // namespace spes_wire
