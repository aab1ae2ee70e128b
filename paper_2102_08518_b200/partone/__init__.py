"""Part-I table producer: spline + lattice -> SplineSpace (sub-region tables,
per-region reference polynomials, stencils).  The reference consumes these
tables but ships only six toy fixtures (pkg/scripts/make_fixtures.py); this
package builds the spaces the benchmark configurations need."""
