"""CPU oracle for parity tests and the CPU baseline (test infrastructure only;
see gmp_oracle.py's header). The product package never imports it."""
