"""CacheBlend fp64 CPU oracle. TEST INFRASTRUCTURE ONLY (see cacheblend_oracle.py header)."""
