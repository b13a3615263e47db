"""CPU oracle -- TEST INFRASTRUCTURE ONLY (see oracle.h).  Never imported by the product path."""
