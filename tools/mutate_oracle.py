"""Mutation check of the oracle pins: each plausible mistake in oracle/oracle.c must fail a
`-m "not gpu"` oracle pin test.  Run: python tools/mutate_oracle.py"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = open(os.path.join(ROOT, "oracle", "oracle.c")).read()

MUTANTS = {
    "flip iono sign": ("return orc_iono_dir(n, fs, fc, tec, -1, method, x, y);", "return orc_iono_dir(n, fs, fc, tec, +1, method, x, y);"),
    "one-way delay": ("return 2.0 * k2 / (ORC_C * f_hz);", "return k2 / (ORC_C * f_hz);"),
    "K2 uses 4 pi^2": ("(8.0 * ORC_PI * ORC_PI * ORC_ME * ORC_EPS0)", "(4.0 * ORC_PI * ORC_PI * ORC_ME * ORC_EPS0)"),
    "Nyquist bin positive": ("(k >= n / 2) ? k - n : k", "(k > n / 2) ? k - n : k"),
    "no fc offset": ("return fc + fs * (double)kk / (double)n;", "return fs * (double)kk / (double)n;"),
    "no 1/n": ("for (int64_t t = 0; t < 2 * n; ++t) y[t] /= (double)n;", ""),
    "fft twiddle sign": ("double ang = (double)sign * 2.0 * ORC_PI * (double)j / (double)len;", "double ang = -(double)sign * 2.0 * ORC_PI * (double)j / (double)len;"),
    "window off by one": ("int64_t k_lo = (int64_t)floor(t - 0.5 * (double)W) + 1;", "int64_t k_lo = (int64_t)floor(t - 0.5 * (double)W);"),
    "resample at alpha": ("double beta = 1.0 / alpha;\n  double L = 0.5 * (double)W;", "double beta = alpha;\n  double L = 0.5 * (double)W;"),
    "carrier sign": ("    double ang = -2.0 * ORC_PI * r;\n    double c = cos(ang), s = sin(ang);\n    y[2 * m] = re * c - im * s;\n    y[2 * m + 1] = re * s + im * c;\n  }\n  return 0;\n}\n\n/* rectangular", "    double ang = 2.0 * ORC_PI * r;\n    double c = cos(ang), s = sin(ang);\n    y[2 * m] = re * c - im * s;\n    y[2 * m + 1] = re * s + im * c;\n  }\n  return 0;\n}\n\n/* rectangular"),
    "sinc missing pi": ("return sin(ORC_PI * d) / (ORC_PI * d);", "return sin(ORC_PI * d) / (d);"),
    "conj multiply": ("X[2 * k + 1] = xr * s + xi * c;", "X[2 * k + 1] = -xr * s + xi * c;"),
    "drop last sample": ("if (k < 0 || k >= n) continue;", "if (k < 0 || k >= n - 1) continue;"),
    "correlate without conj": ("ar += yr * rr + yi * ri; /* y conj(r) */\n      ai += yi * rr - yr * ri;", "ar += yr * rr - yi * ri;\n      ai += yi * rr + yr * ri;"),
    "correlate lag sign": ("const int64_t t = (s + m) % n;", "const int64_t t = (s - m + n) % n;"),
    "compress skips iono": ("int rc = orc_iono(n, fs, fc, tec, (n & (n - 1)) ? 1 : 0, x, y);", "int rc = 0; memcpy(y, x, sizeof(double) * 2 * (size_t)n);"),
    "taper half-width W": ("double L = 0.5 * (double)W;", "double L = (double)W;"),
    "taper not normalised": ("return orc_bessel_i0(kb * sqrt(r)) / orc_bessel_i0(kb);", "return orc_bessel_i0(kb * sqrt(r));"),
    "I0 series (j!) not squared": ("term *= q / ((double)j * (double)j);", "term *= q / (double)j;"),
    "pq no Nyquist split": ("      Y[2 * h] *= 0.5;\n      Y[2 * h + 1] *= 0.5;\n", ""),
    "pq scale 1/M": ("y[2 * m] = (m < M) ? z[2 * m] / (double)n : 0.0;", "y[2 * m] = (m < M) ? z[2 * m] / (double)M : 0.0;"),
    "pq odd length rule": ("return n + 2 * (int64_t)llround(0.5 * ((double)n * alpha - (double)n));", "return n + (int64_t)llround((double)n * alpha - (double)n);"),
    "no u==0 sinc case": ("if (d == 0.0) return 1.0;\n  if (d == floor(d)) return 0.0;", "if (d == 0.0) return 1.0;"),
    "pq carrier sign": ("    double ang = -2.0 * ORC_PI * r;\n    double c = cos(ang), sn = sin(ang);", "    double ang = 2.0 * ORC_PI * r;\n    double c = cos(ang), sn = sin(ang);"),
    "pq carrier from 1/alpha": ("const double beta_eff = (double)n / (double)M;", "const double beta_eff = 1.0 / alpha;"),
    "pq no carrier": ("double psi = fc * (1.0 - beta_eff) * (double)m / fs;", "double psi = 0.0 * fc * (1.0 - beta_eff) * (double)m / fs;"),
    "exact carrier sign": ("    double ang = -2.0 * ORC_PI * r;\n    double c = cos(ang), s = sin(ang);\n    y[2 * m] = re * c - im * s;\n    y[2 * m + 1] = re * s + im * c;\n  }\n  return 0;\n}\n\n/* ---", "    double ang = 2.0 * ORC_PI * r;\n    double c = cos(ang), s = sin(ang);\n    y[2 * m] = re * c - im * s;\n    y[2 * m + 1] = re * s + im * c;\n  }\n  return 0;\n}\n\n/* ---"),
    "exact no carrier": ("    double psi = fc * (1.0 - beta) * (double)m / fs;\n    double r = psi - nearbyint(psi);\n    double ang = -2.0 * ORC_PI * r;\n    double c = cos(ang), s = sin(ang);\n    y[2 * m] = re * c - im * s;\n    y[2 * m + 1] = re * s + im * c;\n  }\n  return 0;\n}\n\n/* ---", "    double psi = 0.0;\n    double r = psi - nearbyint(psi);\n    double ang = -2.0 * ORC_PI * r;\n    double c = cos(ang), s = sin(ang);\n    y[2 * m] = re * c - im * s;\n    y[2 * m + 1] = re * s + im * c;\n  }\n  return 0;\n}\n\n/* ---"),
    "pq_at inverse length n": ("const int64_t km = (int64_t)(((__int128)k * m) % M);", "const int64_t km = (int64_t)(((__int128)k * m) % n);"),
    "pq_at forward sign": ("  memcpy(X, x, sizeof(double) * 2 * (size_t)n);\n  orc_fft(n, X, -1);", "  memcpy(X, x, sizeof(double) * 2 * (size_t)n);\n  orc_fft(n, X, +1);"),
    "hann half-width W": ("double orc_hann(double d, double L) { return 0.5 * (1.0 + cos(ORC_PI * d / L)); }", "double orc_hann(double d, double L) { return 0.5 * (1.0 + cos(ORC_PI * d / (2.0 * L))); }"),
    "hann not halved": ("double orc_hann(double d, double L) { return 0.5 * (1.0 + cos(ORC_PI * d / L)); }", "double orc_hann(double d, double L) { return (1.0 + cos(ORC_PI * d / L)); }"),
}

failed_to_catch = []
with tempfile.TemporaryDirectory() as d:
    for name, (a, b) in [(k, v) for k, v in MUTANTS.items() if len(sys.argv) < 2 or k in sys.argv[1:]]:
        assert a in SRC, name
        src = os.path.join(d, "m.c")
        lib = os.path.join(d, "m.so")
        open(src, "w").write(SRC.replace(a, b, 1))
        if os.path.exists(lib):
            os.remove(lib)
        env = dict(os.environ, DISPCORR_ORACLE_SRC=src, DISPCORR_ORACLE_LIB=lib)
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "tests/test_oracle_pins.py"], cwd=ROOT, env=env,
                           capture_output=True, text=True, timeout=300)
        caught = r.returncode != 0
        print(f"{'CAUGHT ' if caught else 'MISSED '} {name}")
        if not caught:
            failed_to_catch.append(name)
print("all mutants caught" if not failed_to_catch else f"missed: {failed_to_catch}")
sys.exit(1 if failed_to_catch else 0)
