// gmpxx.h — minimal test-infrastructure shim over the runtime libgmp.so.10.
//
// ORACLE / TEST INFRASTRUCTURE ONLY. This image ships libgmp.so.10 but no GMP
// headers, so the reference verifier (/root/reference/proj) cannot be compiled
// as-is. This header declares the handful of GMP C entry points the reference
// uses (struct layout per the GMP 6.x ABI: {int alloc; int size; limb* d}) and
// wraps them in value-semantic mpz_class / mpq_class types with the operator
// surface the reference's headers and sources need (interval.hpp, decimal.cpp,
// gen.cpp, model_io.cpp, oracle.hpp). Operators return plain values instead
// of gmpxx expression templates; comparisons return bool.
//
// Never linked into the product library.
#pragma once

#include <cstddef>
#include <cstdlib>
#include <string>
#include <utility>

extern "C" {
typedef unsigned long mp_limb_t;
typedef struct {
  int _mp_alloc;
  int _mp_size;
  mp_limb_t* _mp_d;
} __mpz_struct;
typedef struct {
  __mpz_struct _mp_num;
  __mpz_struct _mp_den;
} __mpq_struct;

void __gmpz_init(__mpz_struct*);
void __gmpz_clear(__mpz_struct*);
void __gmpz_set(__mpz_struct*, const __mpz_struct*);
void __gmpz_set_si(__mpz_struct*, long);
int __gmpz_set_str(__mpz_struct*, const char*, int);
char* __gmpz_get_str(char*, int, const __mpz_struct*);
void __gmpz_add(__mpz_struct*, const __mpz_struct*, const __mpz_struct*);
void __gmpz_sub(__mpz_struct*, const __mpz_struct*, const __mpz_struct*);
void __gmpz_mul(__mpz_struct*, const __mpz_struct*, const __mpz_struct*);
void __gmpz_tdiv_q(__mpz_struct*, const __mpz_struct*, const __mpz_struct*);
void __gmpz_tdiv_r(__mpz_struct*, const __mpz_struct*, const __mpz_struct*);
void __gmpz_neg(__mpz_struct*, const __mpz_struct*);
int __gmpz_cmp(const __mpz_struct*, const __mpz_struct*);

void __gmpq_init(__mpq_struct*);
void __gmpq_clear(__mpq_struct*);
void __gmpq_set(__mpq_struct*, const __mpq_struct*);
void __gmpq_set_d(__mpq_struct*, double);
double __gmpq_get_d(const __mpq_struct*);
void __gmpq_set_num(__mpq_struct*, const __mpz_struct*);
void __gmpq_set_den(__mpq_struct*, const __mpz_struct*);
void __gmpq_get_num(__mpz_struct*, const __mpq_struct*);
void __gmpq_get_den(__mpz_struct*, const __mpq_struct*);
void __gmpq_canonicalize(__mpq_struct*);
void __gmpq_add(__mpq_struct*, const __mpq_struct*, const __mpq_struct*);
void __gmpq_sub(__mpq_struct*, const __mpq_struct*, const __mpq_struct*);
void __gmpq_mul(__mpq_struct*, const __mpq_struct*, const __mpq_struct*);
void __gmpq_div(__mpq_struct*, const __mpq_struct*, const __mpq_struct*);
void __gmpq_neg(__mpq_struct*, const __mpq_struct*);
void __gmpq_abs(__mpq_struct*, const __mpq_struct*);
int __gmpq_cmp(const __mpq_struct*, const __mpq_struct*);
}

class mpz_class {
 public:
  __mpz_struct z;
  mpz_class() { __gmpz_init(&z); }
  mpz_class(long v) { __gmpz_init(&z); __gmpz_set_si(&z, v); }
  mpz_class(int v) : mpz_class(static_cast<long>(v)) {}
  mpz_class(const std::string& s, int base) {
    __gmpz_init(&z);
    if (__gmpz_set_str(&z, s.c_str(), base) != 0) __gmpz_set_si(&z, 0);
  }
  mpz_class(const mpz_class& o) { __gmpz_init(&z); __gmpz_set(&z, &o.z); }
  mpz_class(mpz_class&& o) noexcept { __gmpz_init(&z); std::swap(z, o.z); }
  mpz_class& operator=(const mpz_class& o) { if (this != &o) __gmpz_set(&z, &o.z); return *this; }
  mpz_class& operator=(mpz_class&& o) noexcept { std::swap(z, o.z); return *this; }
  ~mpz_class() { __gmpz_clear(&z); }

  std::string get_str(int base = 10) const {
    char* p = __gmpz_get_str(nullptr, base, &z);
    std::string s(p);
    std::free(p);
    return s;
  }
  mpz_class operator-() const { mpz_class r; __gmpz_neg(&r.z, &z); return r; }
  mpz_class& operator*=(const mpz_class& o) { __gmpz_mul(&z, &z, &o.z); return *this; }
  mpz_class& operator/=(const mpz_class& o) { __gmpz_tdiv_q(&z, &z, &o.z); return *this; }
  friend mpz_class operator*(const mpz_class& a, const mpz_class& b) { mpz_class r; __gmpz_mul(&r.z, &a.z, &b.z); return r; }
  friend mpz_class operator+(const mpz_class& a, const mpz_class& b) { mpz_class r; __gmpz_add(&r.z, &a.z, &b.z); return r; }
  friend mpz_class operator-(const mpz_class& a, const mpz_class& b) { mpz_class r; __gmpz_sub(&r.z, &a.z, &b.z); return r; }
  friend mpz_class operator%(const mpz_class& a, const mpz_class& b) { mpz_class r; __gmpz_tdiv_r(&r.z, &a.z, &b.z); return r; }
  friend bool operator==(const mpz_class& a, const mpz_class& b) { return __gmpz_cmp(&a.z, &b.z) == 0; }
  friend bool operator!=(const mpz_class& a, const mpz_class& b) { return __gmpz_cmp(&a.z, &b.z) != 0; }
  friend bool operator<(const mpz_class& a, const mpz_class& b) { return __gmpz_cmp(&a.z, &b.z) < 0; }
  friend bool operator>(const mpz_class& a, const mpz_class& b) { return __gmpz_cmp(&a.z, &b.z) > 0; }
};

class mpq_class {
 public:
  __mpq_struct q;
  mpq_class() { __gmpq_init(&q); }
  mpq_class(long v) { __gmpq_init(&q); set_si(v, 1); }
  mpq_class(int v) : mpq_class(static_cast<long>(v)) {}
  mpq_class(unsigned long v) : mpq_class(static_cast<long>(v)) {}
  mpq_class(long long v) : mpq_class(static_cast<long>(v)) {}
  mpq_class(double d) { __gmpq_init(&q); __gmpq_set_d(&q, d); }
  mpq_class(long n, long d) { __gmpq_init(&q); set_si(n, d); __gmpq_canonicalize(&q); }
  mpq_class(int n, int d) : mpq_class(static_cast<long>(n), static_cast<long>(d)) {}
  mpq_class(long n, int d) : mpq_class(n, static_cast<long>(d)) {}
  mpq_class(int n, long d) : mpq_class(static_cast<long>(n), d) {}
  mpq_class(const mpz_class& n, const mpz_class& d) {
    __gmpq_init(&q);
    __gmpq_set_num(&q, &n.z);
    __gmpq_set_den(&q, &d.z);
  }
  mpq_class(const mpq_class& o) { __gmpq_init(&q); __gmpq_set(&q, &o.q); }
  mpq_class(mpq_class&& o) noexcept { __gmpq_init(&q); std::swap(q, o.q); }
  mpq_class& operator=(const mpq_class& o) { if (this != &o) __gmpq_set(&q, &o.q); return *this; }
  mpq_class& operator=(mpq_class&& o) noexcept { std::swap(q, o.q); return *this; }
  ~mpq_class() { __gmpq_clear(&q); }

  void canonicalize() { __gmpq_canonicalize(&q); }
  double get_d() const { return __gmpq_get_d(&q); }
  mpz_class get_num() const { mpz_class r; __gmpq_get_num(&r.z, &q); return r; }
  mpz_class get_den() const { mpz_class r; __gmpq_get_den(&r.z, &q); return r; }

  mpq_class operator-() const { mpq_class r; __gmpq_neg(&r.q, &q); return r; }
  mpq_class& operator+=(const mpq_class& o) { __gmpq_add(&q, &q, &o.q); return *this; }
  mpq_class& operator-=(const mpq_class& o) { __gmpq_sub(&q, &q, &o.q); return *this; }
  mpq_class& operator*=(const mpq_class& o) { __gmpq_mul(&q, &q, &o.q); return *this; }
  mpq_class& operator/=(const mpq_class& o) { __gmpq_div(&q, &q, &o.q); return *this; }
  friend mpq_class operator+(const mpq_class& a, const mpq_class& b) { mpq_class r; __gmpq_add(&r.q, &a.q, &b.q); return r; }
  friend mpq_class operator-(const mpq_class& a, const mpq_class& b) { mpq_class r; __gmpq_sub(&r.q, &a.q, &b.q); return r; }
  friend mpq_class operator*(const mpq_class& a, const mpq_class& b) { mpq_class r; __gmpq_mul(&r.q, &a.q, &b.q); return r; }
  friend mpq_class operator/(const mpq_class& a, const mpq_class& b) { mpq_class r; __gmpq_div(&r.q, &a.q, &b.q); return r; }
  friend bool operator==(const mpq_class& a, const mpq_class& b) { return __gmpq_cmp(&a.q, &b.q) == 0; }
  friend bool operator!=(const mpq_class& a, const mpq_class& b) { return __gmpq_cmp(&a.q, &b.q) != 0; }
  friend bool operator<(const mpq_class& a, const mpq_class& b) { return __gmpq_cmp(&a.q, &b.q) < 0; }
  friend bool operator>(const mpq_class& a, const mpq_class& b) { return __gmpq_cmp(&a.q, &b.q) > 0; }
  friend bool operator<=(const mpq_class& a, const mpq_class& b) { return __gmpq_cmp(&a.q, &b.q) <= 0; }
  friend bool operator>=(const mpq_class& a, const mpq_class& b) { return __gmpq_cmp(&a.q, &b.q) >= 0; }
  friend mpq_class abs(const mpq_class& a) { mpq_class r; __gmpq_abs(&r.q, &a.q); return r; }

 private:
  void set_si(long n, long d) {
    mpz_class zn(n), zd(d);
    __gmpq_set_num(&q, &zn.z);
    __gmpq_set_den(&q, &zd.z);
  }
};
