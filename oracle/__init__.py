"""TEST INFRASTRUCTURE ONLY: sequential CPU oracle of the DSMC step (see dsmc_oracle.h)."""
