"""Oracle package — TEST INFRASTRUCTURE ONLY (see oracle.py / kw_oracle.c headers)."""
