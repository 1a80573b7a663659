// pk_generic_rt.cuh -- device runtime of the generic program path (generic.py):
// values with the reference interpreter's semantics
// (/root/reference/pkg/src/parakern/interp.py:43-50, 83-125, 189-212), for
// kernels generic.py emits from .mfk programs outside the seven hand-written
// families and compiles with NVRTC (sm_100a).  Not part of libpk.so.
//
// Two value models, chosen per call by the host:
//  * PK_MODE_INT: every value is an int (int64 here).  + - * with an overflow
//    check (the reference's ints are unbounded: a result beyond int64 raises
//    OverflowError instead of wrapping), / and % as C99 truncation (c_div /
//    c_mod, interp.py:43-50).
//  * dynamic: a value is a tagged word -- int, float (binary64), bool, object
//    (an index into the caller's objects: moved unchanged, interp.py:189-206)
//    -- with Python's rules: int op int -> int (exact or OverflowError),
//    anything with a float -> float (the int rounded to nearest), c_div on
//    floats = CPython's float floor division of the absolute values with the
//    sign (float_divmod), exact int/float comparison.
// Errors (first one wins, the host raises the matching exception): index out
// of range -> IndexError, zero divisor -> ZeroDivisionError, int beyond int64
// -> OverflowError, float index / arithmetic on an object -> TypeError, a
// local read before any assignment -> KeyError.
#pragma once

#define PK_E_INDEX 1
#define PK_E_ZERO 2
#define PK_E_OVERFLOW 3
#define PK_E_TYPE 4
#define PK_E_KEY 5
#define PK_E_WIDEN 6  // a value stored into 32-bit words does not fit: the host reruns on 64-bit words

typedef long long i64;
typedef unsigned long long u64;

struct PkErr {
    int code;
    int pad;
    i64 info[3];
};

__device__ __forceinline__ void pk_fail(PkErr *e, int code, i64 a, i64 b, i64 c) {
    if (atomicCAS(&e->code, 0, -1) == 0) {  // claim, fill, publish
        e->info[0] = a;
        e->info[1] = b;
        e->info[2] = c;
        __threadfence();
        atomicExch(&e->code, code);
    }
}

// ---- int64 with the reference's unbounded-int results (or OverflowError) ----
__device__ __forceinline__ i64 pk_iadd(PkErr *e, i64 a, i64 b) {
    const i64 r = (i64)((u64)a + (u64)b);
    if (((a ^ r) & (b ^ r)) < 0) pk_fail(e, PK_E_OVERFLOW, 0, 0, 0);
    return r;
}
__device__ __forceinline__ i64 pk_isub(PkErr *e, i64 a, i64 b) {
    const i64 r = (i64)((u64)a - (u64)b);
    if (((a ^ b) & (a ^ r)) < 0) pk_fail(e, PK_E_OVERFLOW, 0, 0, 0);
    return r;
}
__device__ __forceinline__ i64 pk_imul(PkErr *e, i64 a, i64 b) {
    const i64 lo = (i64)((u64)a * (u64)b);
    const i64 hi = __mul64hi(a, b);
    if (hi != (lo >> 63)) pk_fail(e, PK_E_OVERFLOW, 0, 0, 0);
    return lo;
}
// c_div: |a| // |b|, negated when the signs differ (truncation toward zero)
__device__ __forceinline__ i64 pk_idiv(PkErr *e, i64 a, i64 b) {
    if (b == 0) {
        pk_fail(e, PK_E_ZERO, 0, 0, 0);
        return 0;
    }
    const u64 ua = a < 0 ? (u64)0 - (u64)a : (u64)a, ub = b < 0 ? (u64)0 - (u64)b : (u64)b;
    const u64 q = ua / ub;
    if ((a >= 0) == (b >= 0)) {
        if (q > (u64)0x7fffffffffffffffULL) pk_fail(e, PK_E_OVERFLOW, 0, 0, 0);
        return (i64)q;
    }
    return (i64)((u64)0 - q);
}
// c_mod(a, b) = a - b * c_div(a, b)
__device__ __forceinline__ i64 pk_imod(PkErr *e, i64 a, i64 b) {
    const i64 q = pk_idiv(e, a, b);
    return b == 0 ? 0 : pk_isub(e, a, pk_imul(e, b, q));
}

// ---- CPython float floor division (float_divmod) of non-negative operands ----
__device__ __forceinline__ double pk_floordiv(double x, double y) {
    const double mod = fmod(x, y);
    const double div = __ddiv_rn(__dsub_rn(x, mod), y);
    if (div != 0.0) {
        double fl = floor(div);
        if (__dsub_rn(div, fl) > 0.5) fl = __dadd_rn(fl, 1.0);
        return fl;
    }
    return copysign(0.0, __ddiv_rn(x, y));
}

#ifndef PK_MODE_INT
// ---- dynamic values ----
#define PK_T_INT 0
#define PK_T_FLOAT 1
#define PK_T_BOOL 2
#define PK_T_OBJ 3
#define PK_T_UNDEF 4

struct V {
    i64 i;     // int / bool value, object index
    double f;  // float value
    int t;
};
struct PV {  // array element in device memory: 8 value bytes + the tag
    i64 bits;
    int t;
    int pad;
};

__device__ __forceinline__ V vi(i64 x) { V v; v.i = x; v.f = 0.0; v.t = PK_T_INT; return v; }
__device__ __forceinline__ V vf(double x) { V v; v.i = 0; v.f = x; v.t = PK_T_FLOAT; return v; }
__device__ __forceinline__ V vundef() { V v; v.i = 0; v.f = 0.0; v.t = PK_T_UNDEF; return v; }
__device__ __forceinline__ bool v_isint(const V &a) { return a.t == PK_T_INT || a.t == PK_T_BOOL; }
__device__ __forceinline__ double v_asf(const V &a) { return a.t == PK_T_FLOAT ? a.f : __ll2double_rn(a.i); }

__device__ __forceinline__ V pk_unpack(const PV &p) {
    V v;
    v.t = p.t;
    v.i = p.bits;
    v.f = p.t == PK_T_FLOAT ? __longlong_as_double(p.bits) : 0.0;
    return v;
}
__device__ __forceinline__ PV pk_pack(const V &v) {
    PV p;
    p.t = v.t;
    p.pad = 0;
    p.bits = v.t == PK_T_FLOAT ? __double_as_longlong(v.f) : v.i;
    return p;
}

// operands checked: both numbers (else TypeError; an undefined local: KeyError)
__device__ __forceinline__ bool v_num2(PkErr *e, const V &a, const V &b) {
    if (a.t == PK_T_UNDEF || b.t == PK_T_UNDEF) {
        pk_fail(e, PK_E_KEY, 0, 0, 0);
        return false;
    }
    if (a.t == PK_T_OBJ || b.t == PK_T_OBJ) {
        pk_fail(e, PK_E_TYPE, 0, 0, 0);
        return false;
    }
    return true;
}
__device__ __forceinline__ V v_add(PkErr *e, V a, V b) {
    if (!v_num2(e, a, b)) return vi(0);
    if (v_isint(a) && v_isint(b)) return vi(pk_iadd(e, a.i, b.i));
    return vf(__dadd_rn(v_asf(a), v_asf(b)));
}
__device__ __forceinline__ V v_sub(PkErr *e, V a, V b) {
    if (!v_num2(e, a, b)) return vi(0);
    if (v_isint(a) && v_isint(b)) return vi(pk_isub(e, a.i, b.i));
    return vf(__dsub_rn(v_asf(a), v_asf(b)));
}
__device__ __forceinline__ V v_mul(PkErr *e, V a, V b) {
    if (!v_num2(e, a, b)) return vi(0);
    if (v_isint(a) && v_isint(b)) return vi(pk_imul(e, a.i, b.i));
    return vf(__dmul_rn(v_asf(a), v_asf(b)));
}
__device__ __forceinline__ bool v_nonneg(const V &a) { return a.t == PK_T_FLOAT ? a.f >= 0.0 : a.i >= 0; }
__device__ __forceinline__ V v_div(PkErr *e, V a, V b) {
    if (!v_num2(e, a, b)) return vi(0);
    if (v_isint(a) && v_isint(b)) return vi(pk_idiv(e, a.i, b.i));
    const double y = fabs(v_asf(b));
    if (y == 0.0) {
        pk_fail(e, PK_E_ZERO, 0, 0, 0);
        return vi(0);
    }
    const double q = pk_floordiv(fabs(v_asf(a)), y);
    return vf(v_nonneg(a) == v_nonneg(b) ? q : -q);
}
__device__ __forceinline__ V v_mod(PkErr *e, V a, V b) {
    const V q = v_div(e, a, b);
    return v_sub(e, a, v_mul(e, b, q));
}

// exact comparison of an int with a float: -1, 0, 1, or 2 when unordered (NaN)
__device__ __forceinline__ int pk_cmp_if(i64 i, double f) {
    if (f != f) return 2;
    if (i > -(1LL << 53) && i < (1LL << 53)) {  // exact as a double
        const double d = (double)i;
        return d < f ? -1 : (d > f ? 1 : 0);
    }
    if (f >= 9223372036854775808.0) return -1;
    if (f < -9223372036854775808.0) return 1;
    const double fl = floor(f);
    const i64 fi = (i64)fl;
    if (i < fi) return -1;
    if (i > fi) return 1;
    return f > fl ? -1 : 0;
}
// op: 0 <, 1 <=, 2 >, 3 >=, 4 ==, 5 !=
__device__ __forceinline__ bool v_cmp(PkErr *e, int op, V a, V b) {
    if (a.t == PK_T_UNDEF || b.t == PK_T_UNDEF) {
        pk_fail(e, PK_E_KEY, 0, 0, 0);
        return false;
    }
    if (a.t == PK_T_OBJ || b.t == PK_T_OBJ) {
        // an object equals only itself here; ordering an object raises
        if (op == 4 || op == 5) {
            if (a.t == PK_T_OBJ && b.t == PK_T_OBJ && a.i != b.i) {
                pk_fail(e, PK_E_TYPE, 1, 0, 0);  // equality of two distinct objects: not decidable here
                return false;
            }
            const bool eq = a.t == b.t && a.i == b.i;
            return op == 4 ? eq : !eq;
        }
        pk_fail(e, PK_E_TYPE, 0, 0, 0);
        return false;
    }
    int c;
    if (v_isint(a) && v_isint(b)) {
        c = a.i < b.i ? -1 : (a.i > b.i ? 1 : 0);
    } else if (a.t == PK_T_FLOAT && b.t == PK_T_FLOAT) {
        c = (a.f != a.f || b.f != b.f) ? 2 : (a.f < b.f ? -1 : (a.f > b.f ? 1 : 0));
    } else if (a.t == PK_T_FLOAT) {
        c = pk_cmp_if(b.i, a.f);
        c = c == 2 ? 2 : -c;
    } else {
        c = pk_cmp_if(a.i, b.f);
    }
    if (c == 2) return op == 5;  // NaN: only != holds
    switch (op) {
        case 0: return c < 0;
        case 1: return c <= 0;
        case 2: return c > 0;
        case 3: return c >= 0;
        case 4: return c == 0;
        default: return c != 0;
    }
}
// a subscript: an int (or bool); a float or an object raises TypeError
__device__ __forceinline__ i64 v_index(PkErr *e, const V &a) {
    if (a.t == PK_T_UNDEF) {
        pk_fail(e, PK_E_KEY, 0, 0, 0);
        return -1;
    }
    if (!v_isint(a)) {
        pk_fail(e, PK_E_TYPE, 2, 0, 0);
        return -1;
    }
    return a.i;
}
// a loop bound: range(bound) takes ints only
__device__ __forceinline__ i64 v_bound(PkErr *e, const V &a) { return v_index(e, a); }
// a value stored: an undefined local raises KeyError when read, before the store
__device__ __forceinline__ V v_def(PkErr *e, const V &a) {
    if (a.t == PK_T_UNDEF) pk_fail(e, PK_E_KEY, 0, 0, 0);
    return a;
}

typedef PV Elem;
#define PK_ZERO vi(0)
#define PK_LIT(x) vi(x)
#define PK_LOAD(p) pk_unpack(p)
__device__ __forceinline__ bool pk_store(PkErr *, Elem *d, const V &v) {
    *d = pk_pack(v);
    return true;
}
#else
// ---- every value an int64 (held in int32 words with PK_WORD32) ----
typedef i64 V;
#ifdef PK_WORD32
typedef int Elem;
#else
typedef i64 Elem;
#endif
#define PK_ZERO 0LL
#define PK_LIT(x) (x)
#define PK_LOAD(p) ((i64)(p))
__device__ __forceinline__ bool pk_store(PkErr *e, Elem *d, i64 v) {
#ifdef PK_WORD32
    if (v != (i64)(int)v) {
        pk_fail(e, PK_E_WIDEN, 0, 0, 0);
        return false;
    }
#endif
    *d = (Elem)v;
    (void)e;
    return true;
}
__device__ __forceinline__ V v_add(PkErr *e, V a, V b) { return pk_iadd(e, a, b); }
__device__ __forceinline__ V v_sub(PkErr *e, V a, V b) { return pk_isub(e, a, b); }
__device__ __forceinline__ V v_mul(PkErr *e, V a, V b) { return pk_imul(e, a, b); }
__device__ __forceinline__ V v_div(PkErr *e, V a, V b) { return pk_idiv(e, a, b); }
__device__ __forceinline__ V v_mod(PkErr *e, V a, V b) { return pk_imod(e, a, b); }
__device__ __forceinline__ bool v_cmp(PkErr *, int op, V a, V b) {
    switch (op) {
        case 0: return a < b;
        case 1: return a <= b;
        case 2: return a > b;
        case 3: return a >= b;
        case 4: return a == b;
        default: return a != b;
    }
}
__device__ __forceinline__ i64 v_index(PkErr *, V a) { return a; }
__device__ __forceinline__ i64 v_bound(PkErr *, V a) { return a; }
__device__ __forceinline__ V v_def(PkErr *, V a) { return a; }
__device__ __forceinline__ V vi(i64 x) { return x; }
#endif

// ---- arrays: element buffers with the caller's extents ----
struct PkArr {
    Elem *p;
    i64 rows;  // len(arr)
    i64 cols;  // len(arr[0]) for 2-D arrays, 0 for 1-D
};

// _checked (interp.py:209-212): 0 <= i < len, per subscript
__device__ __forceinline__ bool pk_inb(PkErr *e, int id, const PkArr &a, i64 i, i64 j, int rank) {
    if (i < 0 || i >= a.rows || (rank == 2 && (j < 0 || j >= a.cols))) {
        pk_fail(e, PK_E_INDEX, id, i, j);
        return false;
    }
    return true;
}
__device__ __forceinline__ V pk_ld(PkErr *e, int id, const PkArr &a, i64 i, i64 j, int rank) {
    if (!pk_inb(e, id, a, i, j, rank)) return PK_ZERO;
    return PK_LOAD(a.p[rank == 2 ? i * a.cols + j : i]);
}
__device__ __forceinline__ void pk_st(PkErr *e, int id, const PkArr &a, i64 i, i64 j, int rank, V v) {
    if (!pk_inb(e, id, a, i, j, rank)) return;
    pk_store(e, a.p + (rank == 2 ? i * a.cols + j : i), v);
}
