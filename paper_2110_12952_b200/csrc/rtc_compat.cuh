// rtc_compat.cuh -- the few standard-library pieces the device headers use, so the
// same headers also compile under NVRTC (jit.inc: micro-block kernels specialised
// at run time for descriptors without a built-in wiring).  Under nvcc this is
// just the standard headers.
#pragma once

#ifdef __CUDACC_RTC__
typedef signed char int8_t;
typedef unsigned char uint8_t;
typedef short int16_t;
typedef unsigned short uint16_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef long long int64_t;
typedef unsigned long long uint64_t;
typedef unsigned long long uintptr_t;
#ifndef INT64_MAX
#define INT64_MAX 9223372036854775807LL
#endif

namespace std {
template <class T, T V>
struct integral_constant {
    static constexpr T value = V;
    using value_type = T;
    __host__ __device__ constexpr operator T() const { return V; }
};
using true_type = integral_constant<bool, true>;
using false_type = integral_constant<bool, false>;
template <class A, class B> struct is_same : false_type {};
template <class A> struct is_same<A, A> : true_type {};
template <class T, T... Is> struct integer_sequence { static constexpr int size() { return sizeof...(Is); } };
template <int N, int... Is>
struct make_int_seq_impl : make_int_seq_impl<N - 1, N - 1, Is...> {};
template <int... Is>
struct make_int_seq_impl<0, Is...> { using type = integer_sequence<int, Is...>; };
template <class T, T N>  // (int sequences only)
using make_integer_sequence = typename make_int_seq_impl<N>::type;
}  // namespace std
#else
#include <cstdint>
#include <type_traits>
#include <utility>
#include <cuda_runtime.h>
#endif
