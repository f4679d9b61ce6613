"""The shared seeded generator (inputs/): determinism, known bit patterns, ranges."""
import numpy as np

from inputs import (TINY, MIXTRAL, bf16_bits_to_f32, f32_to_bf16_bits, gen_prompt, splitmix64,
                    stream_u24, uniform_pm1, weight_fp32, tensor_id, KIND_W1)


def test_splitmix64_reference_values():
    # splitmix64 reference outputs for seed 0 (Vigna's splitmix64.c: state += golden, mix)
    assert splitmix64(0) == 0xE220A8397B1DCDAF
    arr = splitmix64(np.array([0, 1], dtype=np.uint64))
    assert int(arr[0]) == 0xE220A8397B1DCDAF
    assert int(arr[1]) == splitmix64(1)


def test_stream_block_independence():
    a = stream_u24(7, 123, 1000)
    b = np.concatenate([stream_u24(7, 123, 400), stream_u24(7, 123, 600, start=400)])
    assert np.array_equal(a, b)
    assert a.max() < (1 << 24)


def test_uniform_symmetric_exact():
    v = uniform_pm1(1, 2, 100000)
    assert v.dtype == np.float32
    assert np.all(np.abs(v) < 1) and np.all(v != 0)
    # odd multiples of 2^-24
    k = (v.astype(np.float64) * 2 ** 24)
    assert np.all(k == np.round(k)) and np.all(np.mod(k, 2) == 1)
    assert abs(float(v.mean())) < 0.01


def test_bf16_rne():
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -2.5, 1.0 + 2 ** -9], dtype=np.float32)
    b = f32_to_bf16_bits(x)
    # 1+2^-8 is a tie between 1 and 1+2^-7 -> even (1.0); 1+3*2^-8 -> 1+2^-6 (even)
    assert bf16_bits_to_f32(b).tolist() == [1.0, 1.0, 1.0 + 2 ** -6, -2.5, 1.0]


def test_weights_scale_and_prompt_range():
    w = weight_fp32(2512, tensor_id(KIND_W1, 3, 5), 64, TINY.d, TINY.d)
    assert np.all(np.abs(w) <= 1 / 16)
    p = gen_prompt(MIXTRAL, 1, 512)
    assert p.min() >= 1 and p.max() < MIXTRAL.V and p.dtype == np.int32
    assert np.array_equal(p, gen_prompt(MIXTRAL, 1, 512))
